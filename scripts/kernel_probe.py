"""Standalone timing of every hot kernel at the ResNet-50 layout through the C ABI
(development / evidence tool; also the ncu target: each kernel runs `--reps` times).

K1  cdsgd_quantize        (fp32 g, fp64 residual)                 20.25 B/elem
F   cdsgd_fused_round     apply(t-1) from N ranks' codes + quantize(t)
K2  cdsgd_apply_quant     N ranks' codes, W (fp64/fp32), g_next -> W', loc
K3  cdsgd_apply_full      gsum, W, g_next -> W', loc

Prints one JSON line per kernel: avg µs (CUDA events, back to back, inputs > L2), achieved
GB/s from the algorithmic bytes, fraction of MEASURED_PEAKS.json hbm_gbs.

    python scripts/kernel_probe.py [--weights f64] [--nranks 1,4] [--reps 20] [--only K1,F,K2,K3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--weights", default="f64")
    ap.add_argument("--nranks", default="1,4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="K1,F,K2,K3")
    args = ap.parse_args()
    import torch

    from paper_2106_10796_b200 import _lib
    from paper_2106_10796_b200.layout import by_name

    lib = _lib.load()
    torch.cuda.set_device(0)
    layout = by_name(args.layout)
    n, nw = layout.total, layout.n_words
    h = layout.handle().ptr
    dev = torch.device("cuda")
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    wdt = _lib.WEIGHTS[args.weights]
    wb = 8 if args.weights == "f64" else 4
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    gen = torch.Generator(device=dev).manual_seed(0)
    g = 0.3 * torch.randn(n, device=dev, generator=gen)
    g2 = 0.3 * torch.randn(n, device=dev, generator=gen)
    r = [torch.zeros(n, dtype=torch.float64, device=dev), torch.zeros(n, dtype=torch.float64, device=dev)]
    W = torch.randn(n, device=dev, generator=gen).to(torch.float64 if wdt else torch.float32)
    loc = torch.empty(n, device=dev)
    err = torch.full((2,), -1, dtype=torch.int64, device=dev)
    gn = torch.zeros(1, dtype=torch.float64, device=dev)
    only = set(args.only.split(","))

    def timeit(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return 1e3 * e0.elapsed_time(e1) / reps

    def report(name, nr, us, nbytes):
        gbs = nbytes / us / 1e3
        print(json.dumps({"kernel": name, "nranks": nr, "weights": args.weights, "layout": args.layout, "n": n,
                          "avg_us": round(us, 2), "bytes": nbytes, "bytes_per_elem": round(nbytes / n, 3),
                          "achieved_gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / peak, 4)}), flush=True)

    words = torch.zeros(nw, dtype=torch.int32, device=dev).view(torch.uint32)
    lib.cdsgd_quantize(h, g.data_ptr(), _lib.F32, r[0].data_ptr(), r[1].data_ptr(), words.data_ptr(), 0.5,
                       err.data_ptr(), 0, st())
    if "K1" in only:
        us = timeit(lambda: lib.cdsgd_quantize(h, g.data_ptr(), _lib.F32, r[1].data_ptr(), r[0].data_ptr(),
                                               words.data_ptr(), 0.5, err.data_ptr(), 0, st()), args.reps)
        report("K1 quantize", 1, us, 20 * n + 4 * nw)
    for nr in [int(x) for x in args.nranks.split(",")]:
        gath = torch.randint(0, 3, (nr * nw,), dtype=torch.int32, device=dev) * 0x5555  # valid codes only
        gath = gath.view(torch.uint32)
        if "F" in only:
            us = timeit(lambda: lib.cdsgd_fused_round(h, g.data_ptr(), r[0].data_ptr(), r[1].data_ptr(), _lib.F64,
                                                      words.data_ptr(), 0.5, err.data_ptr(), 0, W.data_ptr(), wdt,
                                                      loc.data_ptr(), gath.data_ptr(), nr, nw, 0.1, 0.4, 0,
                                                      gn.data_ptr(), st()), args.reps)
            report("F fused_round", nr, us, 4 * n + 16 * n + 2 * wb * n + 4 * n + nr * 4 * nw + 4 * nw)
        if "K2" in only:
            us = timeit(lambda: lib.cdsgd_apply_quant(h, W.data_ptr(), wdt, gath.data_ptr(), nr, nw, 0.5, 0.1,
                                                      g2.data_ptr(), loc.data_ptr(), 0.4, err.data_ptr(), 0,
                                                      gn.data_ptr(), st()), args.reps)
            report("K2 apply_quant", nr, us, 2 * wb * n + 8 * n + nr * 4 * nw)
        if "K3" in only:
            us = timeit(lambda: lib.cdsgd_apply_full(W.data_ptr(), wdt, g.data_ptr(), nr, n, 0.1, g2.data_ptr(),
                                                     loc.data_ptr(), 0.4, None, 0, gn.data_ptr(), st()), args.reps)
            report("K3 apply_full", nr, us, 2 * wb * n + 12 * n)
    e = [int(x) for x in err.cpu().tolist()]
    assert e == [-1, -1], e


if __name__ == "__main__":
    main()
