"""Peer-memory bandwidth calibration on symmetric memory (development tool, torchrun).

Times torch copy kernels that read from / write to a peer's symmetric buffer, and a
cudaMemcpy-style peer copy, at the size of one ResNet-50 stage shard."""

import json
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = 25557032 // world * world
    buf = symm_mem.empty(n, dtype=torch.float32, device="cuda")
    buf.fill_(rank)
    h = symm_mem.rendezvous(buf, dist.group.WORLD)
    peer = (rank + 1) % world
    pv = h.get_buffer(peer, (n,), torch.float32)
    loc = torch.empty(n, device="cuda")
    dist.barrier()
    res = {}
    nb = 4 * n
    res["read_peer_GBs"] = nb / timeit(lambda: loc.copy_(pv)) / 1e3
    dist.barrier()
    res["write_peer_GBs"] = nb / timeit(lambda: pv.copy_(loc)) / 1e3
    dist.barrier()
    res["local_copy_GBs"] = 2 * nb / timeit(lambda: loc.copy_(buf)) / 1e3
    dist.barrier()
    # all peers at once: read a 1/world shard from every rank (the reduce pattern)
    sh = n // world
    views = [h.get_buffer(r, (n,), torch.float32)[rank * sh:(rank + 1) * sh] for r in range(world)]
    acc = torch.empty(sh, device="cuda")

    def red():
        acc.copy_(views[0])
        for v in views[1:]:
            acc.add_(v)

    us = timeit(red)
    res["shard_reduce_remote_GBs"] = (world - 1) * 4 * sh / us / 1e3
    res["shard_reduce_us"] = us
    if rank == 0:
        print(json.dumps({"world": world, "n": n, **{k: round(v, 1) for k, v in res.items()}}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
