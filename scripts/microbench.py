"""Kernel microbenchmarks (development tool): each kernel launched back-to-back,
CUDA-event timed, on ResNet-50-sized buffers, against a torch copy of the same
byte count. Not part of the bench contract."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2106_10796_b200 import _lib  # noqa: E402
from paper_2106_10796_b200.layout import by_name  # noqa: E402


def timeit(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    lay = by_name(sys.argv[1] if len(sys.argv) > 1 else "resnet50")
    n, nw = lay.total, lay.n_words
    lib = _lib.load()
    h = lay.handle().ptr
    st = torch.cuda.current_stream().cuda_stream
    g = 0.3 * torch.randn(n, device="cuda")
    r = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    words = torch.empty(nw, dtype=torch.int32, device="cuda")
    out = {}
    kbytes = 20 * n + 4 * nw
    state = {"i": 0}

    def q_pingpong():
        i = state["i"]
        lib.cdsgd_quantize(h, g.data_ptr(), 0, r[i].data_ptr(), r[i ^ 1].data_ptr(), words.data_ptr(), 0.5, None, 0, st)
        state["i"] ^= 1

    def q_inplace():
        lib.cdsgd_quantize(h, g.data_ptr(), 0, r[0].data_ptr(), r[0].data_ptr(), words.data_ptr(), 0.5, None, 0, st)

    for name, fn in (("quant_pingpong", q_pingpong), ("quant_inplace", q_inplace)):
        us = timeit(fn)
        out[name] = {"us": us, "GBs": kbytes / us / 1e3}
    # torch reference copies with the same bytes
    a = torch.empty(kbytes // 2 // 4, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    us = timeit(lambda: b.copy_(a))
    out["torch_copy_same_bytes"] = {"us": us, "GBs": 2 * a.numel() * 4 / us / 1e3}
    big = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    big2 = torch.empty_like(big)
    us = timeit(lambda: big2.copy_(big), reps=10)
    out["torch_copy_2GiB"] = {"us": us, "GBs": 2 * big.numel() * 2 / us / 1e3}
    # fp64 r-stream alone: r_out = r_in (torch) to see 8-byte stream efficiency
    us = timeit(lambda: r[1].copy_(r[0]))
    out["torch_copy_fp64_r"] = {"us": us, "GBs": 16 * n / us / 1e3}
    W = torch.randn(n, device="cuda")
    gs = torch.randn(n, device="cuda")
    loc = torch.empty(n, device="cuda")
    us = timeit(lambda: lib.cdsgd_apply_full(W.data_ptr(), 0, gs.data_ptr(), 1, n, 0.1, g.data_ptr(), loc.data_ptr(),
                                             0.4, None, 0, None, st))
    out["apply_full"] = {"us": us, "GBs": 20 * n / us / 1e3}
    gath = torch.zeros(nw, dtype=torch.int32, device="cuda")
    us = timeit(lambda: lib.cdsgd_apply_quant(h, W.data_ptr(), 0, gath.data_ptr(), 1, nw, 0.5, 0.1, g.data_ptr(),
                                              loc.data_ptr(), 0.4, None, 0, None, st))
    out["apply_quant_n1"] = {"us": us, "GBs": (16 * n + 4 * nw) / us / 1e3}
    print(json.dumps({k: {kk: round(vv, 1) for kk, vv in v.items()} for k, v in out.items()}, indent=1))


if __name__ == "__main__":
    main()
