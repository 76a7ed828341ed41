"""Host-side cost of CDSGDWorker.step on a small layout (development tool): CPU time per
call vs device time per step, to tell launch-bound from GPU-bound."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10796_b200 import _lib  # noqa: E402
from paper_2106_10796_b200.engine import HyperParams  # noqa: E402
from paper_2106_10796_b200.layout import by_name  # noqa: E402
from paper_2106_10796_b200.worker import CDSGDWorker  # noqa: E402

_lib.load()
dev = torch.device("cuda", 0)
for name in ("resnet20", "resnet50"):
    lay = by_name(name)
    n = lay.total
    pool = [0.3 * torch.randn(n, device=dev) for _ in range(2)]
    wk = CDSGDWorker(lay, HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5,
                                      warmup_n=0), torch.zeros(n, device=dev))
    for i in range(20):
        wk.step(pool[i % 2])
    torch.cuda.synchronize()
    steps = 400 if name == "resnet20" else 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(steps):
        wk.step(pool[i % 2])
    e1.record()
    t1 = time.perf_counter()
    e1.synchronize()
    t2 = time.perf_counter()
    # pure C-ABI call cost (no Python checks): engine_step directly
    st = torch.cuda.current_stream().cuda_stream
    ptr = pool[0].data_ptr()
    t3 = time.perf_counter()
    for i in range(steps):
        wk._lib.cdsgd_engine_step(wk._eng, ptr, st)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: host {1e6 * (t1 - t0) / steps:.2f} us/step (API), {1e6 * (t4 - t3) / steps:.2f} us/step (raw ctypes), "
          f"device {1e3 * e0.elapsed_time(e1) / steps:.2f} us/step, wall {1e6 * (t2 - t0) / steps:.2f}")
    wk.close()
