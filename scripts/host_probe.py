"""Host cost per engine step on a launch-bound layout (ResNet-20-sized): the public
CDSGDWorker.step loop vs the bare ctypes call of cdsgd_engine_step with a fixed stream
(wall-clock per call; the GPU round itself is ~3.2 us, so the host is the bound).

    python scripts/host_probe.py
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import by_name
    from paper_2106_10796_b200.worker import CDSGDWorker, _raw_stream

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    layout = by_name("resnet20")
    n = layout.total
    pool = [0.3 * torch.randn(n, device=dev) for _ in range(2)]
    wk = CDSGDWorker(layout, HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5,
                                         warmup_n=0), torch.zeros(n, device=dev))
    out = {}
    N = 4000
    for _ in range(200):
        wk.step(pool[_ % 2])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        wk.step(pool[i % 2])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out["worker_step_us_host"] = 1e6 * (t1 - t0) / N
    out["worker_step_us_wall"] = 1e6 * (t2 - t0) / N
    fn = wk._lib.cdsgd_engine_step
    eng = wk._eng
    st = _raw_stream(0)
    ptrs = [p.data_ptr() for p in pool]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        fn(eng, ptrs[i & 1], st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out["ctypes_step_us_host"] = 1e6 * (t1 - t0) / N
    out["ctypes_step_us_wall"] = 1e6 * (t2 - t0) / N
    t0 = time.perf_counter()
    for i in range(N):
        _raw_stream(0)
    out["raw_stream_us"] = 1e6 * (time.perf_counter() - t0) / N
    t0 = time.perf_counter()
    for i in range(N):
        wk._lib.cdsgd_launch_count()
    out["ctypes_noop_us"] = 1e6 * (time.perf_counter() - t0) / N
    # the standalone fused-round ABI (same kernel, arguments built per call, no engine state)
    from paper_2106_10796_b200 import _lib

    nw = layout.n_words
    r = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(2)]
    W = torch.zeros(n, dtype=torch.float64, device=dev)
    loc = torch.empty(n, device=dev)
    words = torch.zeros(nw, dtype=torch.int32, device=dev)
    err = torch.full((2,), -1, dtype=torch.int64, device=dev)
    lay = layout.handle().ptr
    ff = wk._lib.cdsgd_fused_round
    args = [(lay, ptrs[i], r[i].data_ptr(), r[i ^ 1].data_ptr(), _lib.F64, words.data_ptr(), 0.5, err.data_ptr(), 0,
             W.data_ptr(), _lib.F64, loc.data_ptr(), words.data_ptr(), 1, nw, 0.1, 0.4, 0, None, st) for i in range(2)]
    for i in range(100):
        ff(*args[i & 1])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        ff(*args[i & 1])
    out["fused_round_abi_us_host"] = 1e6 * (time.perf_counter() - t0) / N
    torch.cuda.synchronize()
    x = torch.zeros(1, device=dev)
    for i in range(100):
        x.add_(1.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        x.add_(1.0)
    out["torch_tiny_kernel_us_host"] = 1e6 * (time.perf_counter() - t0) / N
    torch.cuda.synchronize()
    wk.check()
    wk.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
