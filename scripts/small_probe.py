"""Small-layout latency probe (ResNet-20-sized, BASELINE configs[1]): device time per engine
step with the steps replayed from CUDA graphs of P k-periods, next to the floor of a graph
of back-to-back tiny kernels. Knobs of the engine are read from the environment
(CDSGD_NO_PDL, CDSGD_SMALL_CTAS_PER_SM, CDSGD_CH1_TPW, ...), so run it once per setting:

    CDSGD_SMALL_CTAS_PER_SM=1 python scripts/small_probe.py --periods 1,10

Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def read_probe(n_warps_hint=4096):
    """Phase durations of the fused kernel's last launch, per warp (cycles) and the launch span
    (globaltimer ns): 0/7 = entry/exit globaltimer, 1 entry clock, 2 before the grid-dependency
    wait, 3 after it, 4 a task's loads+compute done, 5 loop done, 6 grad-norm partial done;
    8-11 inside the first task: g, r/W/codes, error word arrived, compute done."""
    import ctypes

    import numpy as np

    from paper_2106_10796_b200 import _lib

    lib = _lib.load()
    P = 16
    buf = np.zeros(n_warps_hint * P, dtype=np.uint64)
    rc = lib.cdsgd_diag_probe(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
    if rc != 0:
        return {"error": rc}
    st = buf.reshape(-1, P).astype(np.int64)
    st = st[st[:, 1] != 0]
    g0, g7 = st[:, 0], st[:, 7]
    t0 = g0.min()
    ph = {"prologue": st[:, 2] - st[:, 1], "wait": st[:, 3] - st[:, 2], "task": st[:, 4] - st[:, 3],
          "loop_rest": st[:, 5] - st[:, 4], "gnorm": st[:, 6] - st[:, 5]}
    if st[:, 8].any():  # first task's phases: error word, g, r/W/codes arrival, compute, packing
        ph.update({"t_p2pchk": st[:, 13] - st[:, 3], "t_loopent": st[:, 14] - st[:, 13], "t_errcodes": st[:, 15] - st[:, 14],
                   "t_ldissue": st[:, 12] - st[:, 15], "t_g": st[:, 8] - st[:, 12], "t_rwc": st[:, 9] - st[:, 8], "t_err": st[:, 10] - st[:, 9],
                   "t_compute": st[:, 11] - st[:, 10], "t_pack": st[:, 4] - st[:, 11]})
    res = {"warps": int(len(st)), "span_ns": int(g7.max() - t0),
           "start_ns": {"p50": float(np.percentile(g0 - t0, 50)), "max": int((g0 - t0).max())},
           "end_ns": {"min": int((g7 - t0).min()), "p50": float(np.percentile(g7 - t0, 50)), "max": int((g7 - t0).max())}}
    for k, v in ph.items():
        res[k + "_cyc"] = {"p10": float(np.percentile(v, 10)), "p50": float(np.percentile(v, 50)),
                           "p90": float(np.percentile(v, 90)), "max": int(v.max())}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="resnet20")
    ap.add_argument("--periods", default="1,10")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--weights", default="f64")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--floor", action="store_true", help="also time a graph of tiny torch kernels")
    ap.add_argument("--tag", default="")
    ap.add_argument("--period", type=int, default=0, help="steps per captured period (default: lcm(k, 2))")
    ap.add_argument("--probe", action="store_true",
                    help="read the fused kernel's phase stamps (a -DCDSGD_PROBE_TIMING build loaded via CDSGD_LIB)")
    args = ap.parse_args()
    import torch

    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import by_name
    from paper_2106_10796_b200.worker import CDSGDWorker

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    layout = by_name(args.layout)
    n = layout.total
    gen = torch.Generator(device=dev).manual_seed(7)
    pool = [0.3 * torch.randn(n, device=dev, generator=gen) for _ in range(2)]
    wk = CDSGDWorker(layout, HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=args.k,
                                         alpha=0.5, warmup_n=0), torch.zeros(n, device=dev), weights=args.weights)
    period = args.period or (args.k if args.k % 2 == 0 else 2 * args.k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"tag": args.tag, "layout": args.layout, "n": n, "k": args.k, "weights": args.weights,
           "env": {k: v for k, v in os.environ.items() if k.startswith("CDSGD_")}, "us_per_step": {}}
    cs = torch.cuda.Stream(dev)
    for P in (int(p) for p in args.periods.split(",")):
        cs.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cs):
            for i in range(period * 4):
                wk.step(pool[i % 2])
        torch.cuda.current_stream(dev).wait_stream(cs)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(period * P):
                wk.step(pool[i % 2])
        reps = max(2, args.reps // P)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        e1.synchronize()
        out["us_per_step"][f"graph_{P}_periods"] = 1e3 * e0.elapsed_time(e1) / (reps * period * P)
        del g
    if args.probe:
        out["probe"] = read_probe(n_warps_hint=4096)
    # host loop through the public API
    torch.cuda.synchronize(dev)
    e0.record()
    for i in range(args.reps * period):
        wk.step(pool[i % 2])
    e1.record()
    e1.synchronize()
    out["us_per_step"]["host_loop"] = 1e3 * e0.elapsed_time(e1) / (args.reps * period)
    wk.check()
    wk.close()
    if args.floor:
        x = torch.zeros(1, device=dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(100):
                x.add_(1.0)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        e1.synchronize()
        out["us_per_tiny_kernel_in_graph"] = 1e3 * e0.elapsed_time(e1) / 5000
    best = min(out["us_per_step"].values())
    out["best_gelem_s"] = n / (best * 1e-6) / 1e9
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
