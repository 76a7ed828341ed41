"""NVLink byte accounting of the fused code exchange (nsys/ncu-free; run under torchrun).

Each rank runs R compressed-only rounds of the engine (k huge, no corrections) on the
ResNet-50 layout with the p2p exchange, where the packed-code all-gather happens inside
the quantizing kernel (NVLink stores to every peer's slot). The NVML data-throughput
counters of every rank's GPU (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, KiB, summed over
links) are read before and after; bytes per round are compared with the algorithmic
(N-1) * P per rank and direction (P = 4 * sum ceil(n_k/16) code bytes), and the in-kernel
exchange bus bandwidth is (N-1) * P over the device time per round.

    torchrun --nproc-per-node 2 scripts/nvlink_probe.py --rounds 200
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def smi_nvlink(idx):
    """Fallback: `nvidia-smi nvlink -gt d` (data throughput counters, KiB per link)."""
    import re
    import subprocess

    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(idx)], capture_output=True, text=True,
                             timeout=30).stdout
    except (OSError, subprocess.TimeoutExpired):
        return None, ""
    tx = sum(int(x) for x in re.findall(r"Tx\w*:\s*(\d+)\s*KiB", out))
    rx = sum(int(x) for x in re.findall(r"Rx\w*:\s*(\d+)\s*KiB", out))
    return ([tx, rx] if (tx or rx) else None), out


def nvlink_kib(handle):
    import pynvml as N

    # scopeId UINT_MAX: summed over every link (a bare field id would read link 0 only)
    fields = [(N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF), (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)]
    try:
        vals = N.nvmlDeviceGetFieldValues(handle, fields)
    except (TypeError, N.NVMLError):
        return None
    out = []
    for v in vals:
        if v.nvmlReturn != 0:
            return None
        out.append(int(v.value.ullVal))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=200)
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--weights", default="f64")
    args = ap.parse_args()
    import pynvml
    import torch
    import torch.distributed as dist

    from paper_2106_10796_b200 import _lib
    from paper_2106_10796_b200.comm import Comm, share_unique_id
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import by_name
    from paper_2106_10796_b200.worker import CDSGDWorker

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    pynvml.nvmlInit()
    # NVML enumerates in PCI order like CUDA by default (CUDA_DEVICE_ORDER unset -> FASTEST_FIRST
    # may differ); match by PCI bus id
    props = torch.cuda.get_device_properties(local)
    bus = None
    if all(hasattr(props, a) for a in ("pci_domain_id", "pci_bus_id", "pci_device_id")):
        bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
    handle = None
    if bus is not None:
        try:
            handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except pynvml.NVMLError:
            handle = None
    if handle is None:
        handle = pynvml.nvmlDeviceGetHandleByIndex(local)
    layout = by_name(args.layout)
    n, nw = layout.total, layout.n_words
    comm = Comm(share_unique_id(rank), world, rank)
    hp = HyperParams(algo="cdsgd", workers=world, eta_global=0.1, eta_local=0.4, k=1 << 30, alpha=0.5, warmup_n=0)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    pool = [0.3 * torch.randn(n, device=dev, generator=gen) for _ in range(2)]
    wk = CDSGDWorker(layout, hp, torch.zeros(n, device=dev), rank=rank, comm=comm, exchange="p2p",
                     weights=args.weights)
    for i in range(10):
        wk.step(pool[i % 2])
    wk.join()
    wk.check()
    dist.barrier(device_ids=[local])
    torch.cuda.synchronize(dev)
    c0 = nvlink_kib(handle)
    s0, raw0 = (None, "")
    if c0 is None:
        s0, raw0 = smi_nvlink(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.rounds):
        wk.step(pool[i % 2])
    wk.join()
    e1.record()
    e1.synchronize()
    c1 = nvlink_kib(handle)
    if c0 is None:
        s1, raw1 = smi_nvlink(local)
        c0, c1 = s0, s1
    ms = e0.elapsed_time(e1)
    wk.check()
    P = 4 * nw
    res = {"rank": rank, "world": world, "rounds": args.rounds, "code_bytes_P": P,
           "expected_bytes_per_round_per_direction": (world - 1) * P, "us_per_round": 1e3 * ms / args.rounds,
           "code_bus_gbs": (world - 1) * P / (ms / args.rounds / 1e3) / 1e9}
    if c0 is not None and c1 is not None:
        tx = (c1[0] - c0[0]) * 1024 / args.rounds
        rx = (c1[1] - c0[1]) * 1024 / args.rounds
        res.update({"nvlink_tx_bytes_per_round": tx, "nvlink_rx_bytes_per_round": rx,
                    "tx_over_expected": tx / ((world - 1) * P), "rx_over_expected": rx / ((world - 1) * P),
                    "nvlink_tx_gbs": tx / (ms / args.rounds / 1e3) / 1e9,
                    "note": "NVML data counters include protocol overhead (flits/headers) and the flag "
                            "traffic; they count every NVLink transfer of the process in the window"})
    else:
        res["nvlink_counters"] = "unavailable (NVML throughput fields and nvidia-smi nvlink -gt d)"
        res["nvidia_smi_nvlink_raw"] = raw0[:600]
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps(allres), flush=True)
    wk.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
