"""Calibrate the paper's time model (Eq. 6-9, paper_2106_10796_b200.costmodel) on B200
(SURVEY §8f rank 4). Run under torchrun, one rank per GPU:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        scripts/calibrate_costmodel.py [--out gpurun_out/costmodel_n4.json]

For each model it MEASURES the four constants with the engine that trains it —
  tau    forward + backward of one iteration (no engine)
  delta  one compressed round on a 1-rank engine (quantize + decode/apply, no exchange)
  psi    a compressed round on the N-rank engine minus delta (the code exchange)
  phi    one full-precision round on the N-rank engine (all-reduce + apply)
— feeds them to the model, and compares its per-algorithm mean iteration time with the
measured iteration time of real training (CDSGDModule, autograd gradients) under each
algorithm. Models: torchvision ResNet-50 (the north-star layout, compute-bound) and a
25.6M-parameter linear layer at batch 8 (communication-bound). Times are CUDA-event
device times, max over ranks.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2106_10796_b200 import _lib, costmodel  # noqa: E402
from paper_2106_10796_b200.comm import Comm, share_unique_id  # noqa: E402
from paper_2106_10796_b200.engine import HyperParams  # noqa: E402
from paper_2106_10796_b200.layout import from_module  # noqa: E402
from paper_2106_10796_b200.model import CDSGDModule  # noqa: E402
from paper_2106_10796_b200.worker import CDSGDWorker  # noqa: E402

K = 4


def timed(fn, iters, warm, world, dev):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def build(name, dev):
    if name == "resnet50":
        import torchvision

        net = torchvision.models.resnet50().to(dev).to(memory_format=torch.channels_last)
        x = torch.randn(64, 3, 224, 224, device=dev).to(memory_format=torch.channels_last)
        y = torch.randint(0, 1000, (64,), device=dev)

        def loss():
            with torch.autocast("cuda", dtype=torch.bfloat16):
                return torch.nn.functional.cross_entropy(net(x), y)
        return net, loss, "torchvision ResNet-50, batch 64, 224x224, bf16 autocast, fp32 weights"
    width = 5056 if name == "wide" else 256  # "wide": 25,563,136 parameters; "tiny": test size
    net = torch.nn.Linear(width, width, bias=False).to(dev)
    x = torch.randn(8, width, device=dev)

    def loss():
        return net(x).square().mean()
    return net, loss, f"Linear({width}, {width}), batch 8 ({width * width:,} parameters, tiny compute)"


def engine_round_time(layout, algo, world, rank, comm, dev, w0):
    """Mean device time of one engine round with a resident gradient (no compute)."""
    hp = HyperParams(algo=algo, workers=world, eta_global=0.01, eta_local=0.01, k=K, alpha=0.5, warmup_n=0)
    wk = CDSGDWorker(layout, hp, w0, rank=rank, comm=comm, device=dev)
    g = [0.01 * torch.randn(layout.total, device=dev) for _ in range(2)]
    state = {"i": 0}

    def step():
        wk.step(g[state["i"] & 1])
        state["i"] += 1
    t = timed(step, 8 * K, 2 * K, world, dev)
    wk.flush()
    wk.close()
    return t


def calibrate(models, world, rank, comm, dev):
    out = {"n_gpus": world, "k": K, "models": {}}
    for name in models:
        torch.manual_seed(0)
        net, loss_fn, desc = build(name, dev)
        layout = from_module(net)
        w0 = torch.cat([p.detach().reshape(-1) for p in net.parameters()])

        def fwd_bwd():
            net.zero_grad(set_to_none=False)
            loss_fn().backward()
        tau = timed(fwd_bwd, 20, 5, world, dev)
        # delta: a compressed round on a 1-rank engine (no exchange) on every GPU
        delta = engine_round_time(layout, "bitsgd", 1, 0, None, dev, w0)
        comp_n = engine_round_time(layout, "bitsgd", world, rank, comm, dev, w0) if world > 1 else delta
        phi = engine_round_time(layout, "ssgd", world, rank, comm, dev, w0) if world > 1 else \
            engine_round_time(layout, "ssgd", 1, 0, None, dev, w0)
        psi = max(comp_n - delta, 0.0)
        p = costmodel.CostParams(tau=tau, phi=phi, psi=min(psi, phi), delta=delta, k=K)
        pred = costmodel.averages(p)
        meas = {}
        for algo in costmodel.ALGOS:
            torch.manual_seed(0)
            net2, loss2, _ = build(name, dev)
            hp = HyperParams(algo=algo, workers=world, eta_global=0.01, eta_local=0.01, k=K, alpha=0.5,
                             warmup_n=0)
            m = CDSGDModule(net2, hp, rank=rank, comm=comm)

            def it():
                loss2().backward()
                m.step()
            meas[algo] = timed(it, 8 * K, 2 * K, world, dev)
            m.flush()
            m.worker.close()
            del m, net2
        out["models"][name] = {
            "workload": desc, "parameters": layout.total, "keys": len(layout),
            "constants_s": {"tau": tau, "phi": phi, "psi": psi, "delta": delta},
            "regime": costmodel.classify_regime(p),
            "predicted_iter_s": pred, "measured_iter_s": meas,
            "measured_over_predicted": {a: meas[a] / pred[a] for a in pred},
            "saving_vs_lusgd_per_iter_s": [costmodel.saving_vs_loc(i, p) for i in range(1, K + 1)],
            "saving_vs_bitsgd_per_iter_s": [costmodel.saving_vs_bit(i, p) for i in range(1, K + 1)],
            "measured_saving_s": {"vs_lusgd": meas["lusgd"] - meas["cdsgd"], "vs_bitsgd": meas["bitsgd"] - meas["cdsgd"]},
        }
        del net
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--models", default="resnet50,wide")
    args = ap.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(
        os.environ.get("LOCAL_RANK", 0))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    comm = Comm(share_unique_id(rank), world, rank) if world > 1 else None
    out = calibrate(args.models.split(","), world, rank, comm, dev)
    if rank == 0:
        s = json.dumps(out, indent=1)
        print(s)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(s)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
