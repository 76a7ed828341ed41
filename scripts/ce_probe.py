"""Copy-engine peer-copy bandwidth on symmetric memory (development tool, torchrun): every
rank copies one shard (n/N fp32) to each peer with cudaMemcpyAsync (copy engines, no SMs),
on one stream or one stream per peer, all ranks at once (the reduce-scatter pattern), alone
and while an HBM-bound kernel runs on the compute stream."""

import json
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = 25557032 // world * world
    sh = n // world
    buf = symm_mem.empty(n, dtype=torch.float32, device="cuda")
    h = symm_mem.rendezvous(buf, dist.group.WORLD)
    src = torch.randn(n, device="cuda")
    peers = [h.get_buffer(r, (n,), torch.float32) for r in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    big = torch.empty(1 << 28, device="cuda")
    big2 = torch.empty_like(big)
    res = {}

    def run(multi, busy):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        for s in streams:
            s.wait_stream(cur)
        if busy:
            big2.copy_(big)  # HBM-bound work on the compute stream meanwhile
        for j, r in enumerate(x for x in range(world) if x != rank):
            st = streams[j] if multi else streams[0]
            with torch.cuda.stream(st):
                peers[r][rank * sh:(rank + 1) * sh].copy_(src[r * sh:(r + 1) * sh], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        e1.record(cur)
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e3

    for name, multi, busy in (("one_stream", False, False), ("stream_per_peer", True, False),
                              ("stream_per_peer_busy", True, True)):
        for _ in range(3):
            run(multi, busy)
        us = sum(run(multi, busy) for _ in range(10)) / 10
        res[name + "_us"] = round(us, 1)
        res[name + "_egress_GBs"] = round((world - 1) * sh * 4 / us / 1e3, 1)
    for _ in range(3):
        big2.copy_(big)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    big2.copy_(big)
    e1.record()
    e1.synchronize()
    res["busy_kernel_alone_us"] = round(e0.elapsed_time(e1) * 1e3, 1)
    if rank == 0:
        print(json.dumps({"world": world, "shard_MB": sh * 4 / 1e6, **res}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
