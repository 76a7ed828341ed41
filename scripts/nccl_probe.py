"""Standalone timing of the exchange collectives through libcdsgd_b200's NCCL comm
(development tool; run under torchrun). Prints per-size time and bus GB/s."""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2106_10796_b200 import _lib  # noqa: E402
from paper_2106_10796_b200.comm import Comm, share_unique_id  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.load()
    comm = Comm(share_unique_id(rank), world, rank)
    res = {}
    for name, n in (("allreduce_resnet50", 25557032), ("allgather_resnet50_words", 1597315)):
        if name.startswith("allreduce"):
            a = torch.randn(n, device="cuda")
            b = torch.empty_like(a)
            fn = lambda: comm.allreduce_sum(a, b)  # noqa: E731
            bus = 2 * (world - 1) / world * 4 * n
        else:
            recv = torch.zeros(world * n, dtype=torch.int32, device="cuda")
            send = recv[rank * n:(rank + 1) * n]
            fn = lambda: comm.allgather_words(send, recv)  # noqa: E731
            bus = (world - 1) * 4 * n
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        res[name] = {"us": round(us, 1), "bus_GBs": round(bus / us / 1e3, 1)}
    if rank == 0:
        print(json.dumps({"world": world, **res}))
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
