import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import torch, numpy as np
from paper_2106_10796_b200.engine import HyperParams
from paper_2106_10796_b200.model import CDSGDModule
from test_gpu_module import net, flat_params
for weights in ("f64","f32"):
  for (bk, pl) in ((1, False), (3, False), (1, True), (3, True)):
    hp = HyperParams(algo="cdsgd", workers=1, eta_global=0.05, eta_local=0.2, k=3, alpha=0.05, warmup_n=2)
    a, b = net(0), net(0)
    ma = CDSGDModule(a, hp, weights=weights); mb = CDSGDModule(b, hp, buckets=bk, pipelined=pl, weights=weights)
    x = torch.randn(64, 3, 8, 8, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)); y = (torch.arange(64, device="cuda") % 5)
    bad = []
    for t in range(4):
        xb, yb = x[t*6:t*6+6], y[t*6:t*6+6]
        torch.nn.functional.cross_entropy(a(xb), yb).backward()
        torch.nn.functional.cross_entropy(b(xb), yb).backward()
        ga = torch.cat([p.grad.reshape(-1) for p in a.parameters()]); gb = torch.cat([p.grad.reshape(-1) for p in b.parameters()]) if not pl else None
        ma.step(); mb.step(); torch.cuda.synchronize()
        pa, pb = flat_params(a), flat_params(b)
        d = [ (n, float(np.abs(pa[s.start:s.start+s.length]-pb[s.start:s.start+s.length]).max())) for n, s in zip(ma.names, ma.layout.spans)]
        bad.append((t, [x for x in d if x[1] > 0], None if gb is None else float((ga-gb).abs().max())))
    print(weights, bk, pl, bad)
