"""Per-stream kernel timeline of the CD-SGD step at N ranks (nsys is not in this image).

torch.profiler (Kineto over CUPTI) records every kernel, memcpy and NCCL call of the
process — including the ones libcdsgd_b200.so launches — with its stream. Each rank
runs `--periods` k-periods of the bench workload inside the profiler, with a
record_function range per engine step; rank 0 writes a Chrome trace
(profiles/<out>.json, open in chrome://tracing or ui.perfetto.dev) and every rank
prints a per-stream summary: busy time per stream, and how much of the exchange
streams' busy time overlaps compute-stream kernels (the paper's compute /
communication overlap).

    torchrun --nproc-per-node 2 scripts/timeline.py --out r2_timeline_n2
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def intervals_union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def overlap(a, b):
    """Total length of the intersection of two interval unions."""
    i = j = 0
    tot = 0.0
    while i < len(a) and j < len(b):
        lo, hi = max(a[i][0], b[j][0]), min(a[i][1], b[j][1])
        if hi > lo:
            tot += hi - lo
        if a[i][1] < b[j][1]:
            i += 1
        else:
            j += 1
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--periods", type=int, default=3)
    ap.add_argument("--exchange", default="p2p")
    ap.add_argument("--out", default="timeline")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from torch.profiler import ProfilerActivity, profile, record_function

    from paper_2106_10796_b200 import _lib
    from paper_2106_10796_b200.comm import Comm, share_unique_id
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import by_name
    from paper_2106_10796_b200.worker import CDSGDWorker

    rank, world, local = (int(os.environ.get(v, d)) for v, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    layout = by_name(args.workload)
    n = layout.total
    comm = Comm(share_unique_id(rank), world, rank) if world > 1 else None
    hp = HyperParams(algo="cdsgd", workers=world, eta_global=0.1, eta_local=0.4, k=args.k, alpha=0.5, warmup_n=0)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    pool = [0.3 * torch.randn(n, device=dev, generator=gen) for _ in range(2)]
    wk = CDSGDWorker(layout, hp, torch.zeros(n, device=dev), rank=rank, comm=comm, exchange=args.exchange)
    for i in range(3 * args.k):
        wk.step(pool[i % 2])
    wk.join()
    wk.check()
    if world > 1:
        dist.barrier(device_ids=[local])
    torch.cuda.synchronize(dev)
    steps = args.periods * args.k
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for i in range(steps):
            t = wk.t
            kind = "compressed" if wk.round_compressed(t) else "correction"
            with record_function(f"cdsgd_step t={t} ({kind})"):
                wk.step(pool[i % 2])
        wk.join()
        torch.cuda.synchronize(dev)
    wk.check()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    trace = os.path.join(ROOT, "gpurun_out", f"{args.out}_rank{rank}.json")
    os.makedirs(os.path.dirname(trace), exist_ok=True)
    prof.export_chrome_trace(trace)
    ev = json.load(open(trace))["traceEvents"]
    by_stream = {}
    names = {}
    for e in ev:
        if e.get("ph") != "X" or e.get("cat") not in ("kernel", "gpu_memcpy", "gpu_memset"):
            continue
        s = e.get("args", {}).get("stream", e.get("tid"))
        by_stream.setdefault(s, []).append((e["ts"], e["ts"] + e["dur"]))
        names.setdefault(s, {}).setdefault(e["name"][:60], 0.0)
        names[s][e["name"][:60]] += e["dur"]
    t0 = min(a for v in by_stream.values() for a, _ in v)
    t1 = max(b for v in by_stream.values() for _, b in v)
    # the compute stream is the one carrying the engine's fused/apply kernels
    def is_compute(s):
        return any(k.startswith(("void cdsgd::k_fused", "void cdsgd::k_apply", "void cdsgd::k_quantize"))
                   for k in names[s])
    comp = [s for s in by_stream if is_compute(s)]
    cu = intervals_union([iv for s in comp for iv in by_stream[s]])
    summary = {"rank": rank, "world": world, "workload": args.workload, "k": args.k, "steps": steps,
               "span_us": t1 - t0, "us_per_step": (t1 - t0) / steps, "streams": {}}
    for s, iv in by_stream.items():
        u = intervals_union(iv)
        busy = sum(b - a for a, b in u)
        top = sorted(names[s].items(), key=lambda kv: -kv[1])[:6]
        summary["streams"][str(s)] = {
            "role": "compute" if s in comp else "exchange",
            "busy_us": busy, "busy_frac": busy / (t1 - t0),
            "overlap_with_compute_us": None if s in comp else overlap(u, cu),
            "top_kernels_us": {k: round(v, 1) for k, v in top}}
    print(json.dumps(summary), flush=True)
    if rank == 0:
        with open(os.path.join(ROOT, "gpurun_out", f"{args.out}_summary.json"), "w") as f:
            json.dump(summary, f, indent=1)
    wk.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
