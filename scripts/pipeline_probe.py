"""Layer-wise pipelining measured on real training: per-iteration device time of
CDSGDModule with buckets = 1 (the round after backward) vs B > 1 (each bucket's round issued
from post-accumulate-grad hooks during backward), next to forward+backward alone. Run under
torchrun (one rank per GPU) or plain python (N=1):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/pipeline_probe.py

Models as scripts/calibrate_costmodel.py: torchvision ResNet-50 (batch 64, bf16 autocast,
fp32 weights) and a 25.6M-parameter linear layer at batch 8 (communication-bound). Exact
mode (fp64 residual and weights), k = 4, CUDA-event time per iteration, max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

from calibrate_costmodel import build, timed  # noqa: E402

from paper_2106_10796_b200 import _lib  # noqa: E402
from paper_2106_10796_b200.comm import Comm, share_unique_id  # noqa: E402
from paper_2106_10796_b200.engine import HyperParams  # noqa: E402
from paper_2106_10796_b200.model import CDSGDModule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="resnet50,wide")
    ap.add_argument("--buckets", default="1,2,4,8")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rank, world, local = (int(os.environ.get(v, d)) for v, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    comm = Comm(share_unique_id(rank), world, rank) if world > 1 else None
    res = {"n_gpus": world, "k": 4, "mode": "exact (fp64 residual + fp64 weights)", "models": {}}
    for name in args.models.split(","):
        torch.manual_seed(0)
        net, loss_fn, desc = build(name, dev)

        def fwd_bwd():
            net.zero_grad(set_to_none=False)
            loss_fn().backward()
        tau = timed(fwd_bwd, 20, 5, world, dev)
        row = {"workload": desc, "fwd_bwd_ms": 1e3 * tau, "iter_ms": {}}
        del net
        for nb in (int(b) for b in args.buckets.split(",")):
            torch.manual_seed(0)
            net2, loss2, _ = build(name, dev)
            hp = HyperParams(algo="cdsgd", workers=world, eta_global=0.01, eta_local=0.01, k=4, alpha=0.5,
                             warmup_n=0)
            m = CDSGDModule(net2, hp, rank=rank, comm=comm, buckets=nb)

            def it():
                loss2().backward()
                m.step()
            t = timed(it, 32, 8, world, dev)
            row["iter_ms"][f"buckets={nb}"] = 1e3 * t
            row["iter_ms"][f"buckets={nb}_overhead_ms"] = 1e3 * (t - tau)
            m.flush()
            m.close()
            del m, net2
            torch.cuda.empty_cache()
        res["models"][name] = row
    if rank == 0:
        print(json.dumps(res), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
