"""NVSwitch multicast (NVLS) calibration via torch symmetric-memory ops (development tool).

Times torch.ops.symm_mem.multimem_all_reduce_ / two_shot_all_reduce_ on a ResNet-50
gradient (fp32, 102 MB) against ncclAllReduce, to decide whether a multimem-based
correction exchange can beat the NCCL ring on this box. Run under torchrun."""

import json
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem


def timeit(fn, reps=10):
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
    n = 25557032 // (4 * world) * (4 * world)
    t = symm_mem.empty(n, dtype=torch.float32, device="cuda")
    t.normal_()
    h = symm_mem.rendezvous(t, dist.group.WORLD)
    gname = dist.group.WORLD.group_name
    res = {"multicast_ptr": int(h.multicast_ptr) != 0}
    for name in ("multimem_all_reduce_", "two_shot_all_reduce_"):
        op = getattr(torch.ops.symm_mem, name, None)
        if op is None:
            continue
        try:
            us = timeit(lambda: op(t, "sum", gname))
            res[name + "_us"] = round(us, 1)
        except Exception as exc:  # noqa: BLE001
            res[name] = f"error: {type(exc).__name__}: {str(exc)[:120]}"
    x = torch.randn(n, device="cuda")
    res["nccl_all_reduce_us"] = round(timeit(lambda: dist.all_reduce(x)), 1)
    if rank == 0:
        print(json.dumps({"world": world, "MB": 4 * n / 1e6, **res}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
