"""Multi-GPU parity check, run under torchrun (one rank per GPU) by tests/test_mgpu.py.

Each rank is one CD-SGD worker with its own synthetic gradient stream; packed
codes are exchanged with ncclAllGather and correction gradients with
ncclAllReduce inside libcdsgd_b200.so. Checked against the lock-step oracle with
the same N workers (engine.py:614-663):
  * this rank's residual bit-exact after every round;
  * this rank's compute weights (loc) and the final W within rtol 1e-5 / atol 1e-6;
  * W replicas bitwise identical on every rank (replicated parameter server);
  * the grad-norm metric per round.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cdsgd_oracle as O  # noqa: E402
from paper_2106_10796_b200 import _lib  # noqa: E402
from paper_2106_10796_b200.comm import Comm, share_unique_id  # noqa: E402
from paper_2106_10796_b200.engine import HyperParams  # noqa: E402
from paper_2106_10796_b200.layout import Layout  # noqa: E402
from paper_2106_10796_b200.worker import CDSGDWorker  # noqa: E402

RTOL, ATOL = 1e-5, 1e-6

CASES = [
    # algo, sizes, k, warmup, iters, alpha
    ("cdsgd", [2_600_000, 513], 4, 0, 7, 0.5),  # whole-tile (CH=4) path of the fused kernel
    ("cdsgd", [1000, 37, 16, 1, 4096], 4, 5, 14, 0.5),
    ("cdsgd", [2048, 513], 2, 0, 9, 0.5),
    ("cdsgd", [777], 3, 1, 9, 0.3),
    ("cdsgd", [300, 300], 1, 2, 6, 0.5),
    ("bitsgd", [640, 7], 5, 5, 5, 0.5),
    ("lusgd", [640, 7], 5, 2, 6, 0.5),
    ("ssgd", [640, 7], 5, 5, 4, 0.5),
    # fewer elements than ranks x 4: empty shards in the copy-engine share of the correction
    ("cdsgd", [5, 3], 2, 0, 6, 0.5),
]


def run_case(case, exchange, comm, rank, world, dev):
    algo, sizes, k, warm, iters, alpha = case
    layout = Layout.from_lengths(sizes)
    n = layout.total
    hp = HyperParams(algo=algo, workers=world, eta_global=0.1, eta_local=0.4, k=k, alpha=alpha, warmup_n=warm)
    w0 = O.synthetic_weights(5, n)
    wk = CDSGDWorker(layout, hp, w0, rank=rank, comm=comm, exchange=exchange)
    orc = O.LockstepOracle(w0.astype(np.float64), sizes, O.OracleHP(algo, world, 0.1, 0.4, k, alpha, warm))
    tag = f"{exchange}/{algo} rank {rank}"
    for t in range(iters):
        np.testing.assert_allclose(wk.compute_weights().cpu().numpy(), orc.compute_weights(rank), rtol=RTOL,
                                   atol=ATOL, err_msg=f"{tag} compute weights round {t}")
        grads = [O.synthetic_grad(5, t, w, n) for w in range(world)]
        wk.step(torch.from_numpy(grads[rank]).to(dev))
        orc.step(grads)
        res = wk.residual.cpu().numpy()
        assert np.array_equal(res.view(np.uint64), orc.workers[rank].residual.view(np.uint64)), \
            f"{tag} residual round {t}"
        if orc.compressed[t]:  # this rank's codes of the round, as the engine exposes them
            got = np.concatenate([p.words.cpu().numpy() for p in wk.round_payloads(t)])
            assert np.array_equal(got, orc.words[(t, rank)]), f"{tag} codes round {t}"
    wk.flush()
    W = wk.weights
    np.testing.assert_allclose(W.cpu().numpy(), orc.W, rtol=RTOL, atol=ATOL, err_msg=f"{tag} W")
    allW = [torch.empty_like(W) for _ in range(world)]
    dist.all_gather(allW, W)
    for w in range(world):
        assert torch.equal(allW[w], W), f"{tag}: W replica of rank {w} differs"
    for t in range(iters):
        assert abs(wk.grad_norm(t) - orc.grad_norms[t]) <= 1e-5 * max(1.0, orc.grad_norms[t]), (tag, t)
    wk.close()


def run_pipelined_case(exchange, comm, rank, world, dev):
    """the overlapped paths under real concurrency with caller kernels. An 8.4M-
    element layout (so the default copy-engine share of the correction all-reduce is on),
    k=4, 12 rounds issued back to back with NO host sync between them and a caller compute
    kernel (a matmul) on the same stream between steps — then flush and compare: residual
    bitwise and W within tolerance against the C restatement over EVERY element, W
    replicas bitwise across ranks."""
    from oracle import cpu_port

    sizes = [8_388_608, 4099, 33]
    layout = Layout.from_lengths(sizes)
    n, T = layout.total, 12
    hp = HyperParams(algo="cdsgd", workers=world, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5, warmup_n=0)
    w0 = O.synthetic_weights(8, n)
    grads = [torch.from_numpy(O.synthetic_grad(8, t, rank, n)).to(dev) for t in range(T)]
    a = torch.randn(2048, 2048, device=dev)
    wk = CDSGDWorker(layout, hp, w0, rank=rank, comm=comm, exchange=exchange)
    torch.cuda.synchronize(dev)
    for t in range(T):
        for _ in range(4):
            a = torch.tanh(a @ a * 1e-3)  # caller compute on the same stream, between rounds
        wk.step(grads[t])
    wk.flush()
    W = wk.weights.clone()
    allW = [torch.empty_like(W) for _ in range(world)]
    dist.all_gather(allW, W)
    for w in range(world):
        assert torch.equal(allW[w], W), f"{exchange}: W replica of rank {w} differs (pipelined)"
    if cpu_port.load() is None:
        return
    port = cpu_port.CPortEngine(w0.astype(np.float64), sizes, world, k=4, alpha=0.5)
    for t in range(T):
        port.step(np.stack([O.synthetic_grad(8, t, w, n) for w in range(world)]))
    assert np.array_equal(wk.residual.cpu().numpy().view(np.uint64), port.res[rank].view(np.uint64)), \
        f"{exchange} rank {rank}: residual (pipelined)"
    np.testing.assert_allclose(W.cpu().numpy(), port.W, rtol=RTOL, atol=ATOL, err_msg=f"{exchange} W (pipelined)")
    wk.close()


def run_records_case(exchange, comm, rank, world, dev):
    """World 2: per-round records (records.Recorder) vs the reference's own metrics.csv
    (tests/golden/metrics_n2.csv, unmodified reference: make_metrics_golden.py)."""
    from paper_2106_10796_b200.records import Recorder, read_metrics_csv

    sizes, seed, k, warm, iters = [640, 7, 33], 4, 3, 1, 11
    layout = Layout.from_lengths(sizes)
    n = layout.total
    hp = HyperParams(algo="cdsgd", workers=world, eta_global=0.1, eta_local=0.4, k=k, alpha=0.5, warmup_n=warm)
    wk = CDSGDWorker(layout, hp, O.synthetic_weights(seed, n), rank=rank, comm=comm, exchange=exchange)
    rec = Recorder(wk, batches_per_epoch=1)
    for t in range(iters):
        wk.step(torch.from_numpy(O.synthetic_grad(seed, t, rank, n)).to(dev))
        rec.record(0.0)
    wk.flush()
    mine = rec.records()
    gold = read_metrics_csv(os.path.join(ROOT, "tests", "golden", "metrics_n2.csv"))
    assert len(mine) == len(gold) == iters
    for g, m in zip(gold, mine):
        assert (g.iteration, g.epoch, g.train_loss, g.bytes_pushed, g.compressed) == \
               (m.iteration, m.epoch, m.train_loss, m.bytes_pushed, m.compressed), (g, m)
        assert abs(g.grad_norm - m.grad_norm) <= 1e-6 * g.grad_norm, (exchange, g, m)
    wk.close()


def run_failure_case(exchange, comm, rank, world, dev):
    """Rank world-1 hits a non-finite gradient at round 2 (a compressed round): it raises
    CodecNumericError(round 2) with its residual rolled back, every other rank raises
    PeerFailedError (its flags arrived poisoned) instead of applying the failing rank's
    codes — and nobody hangs or times out."""
    from paper_2106_10796_b200.codec import CodecNumericError

    sizes = [4096, 100]
    layout = Layout.from_lengths(sizes)
    n = layout.total
    hp = HyperParams(algo="cdsgd", workers=world, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5, warmup_n=0)
    wk = CDSGDWorker(layout, hp, O.synthetic_weights(9, n), rank=rank, comm=comm, exchange=exchange)
    bad = rank == world - 1
    for t in range(7):
        g = torch.from_numpy(O.synthetic_grad(9, t, rank, n)).to(dev)
        if bad and t == 2:
            g[4096 + 17] = float("nan")
        wk.step(g)
    try:
        wk.check()
        raise AssertionError(f"rank {rank}: no error reported")
    except CodecNumericError as exc:
        assert bad and (exc.round, exc.key, exc.index) == (2, 1, 17), (rank, exc.round, exc.key, exc.index)
    except _lib.PeerFailedError:
        assert not bad, f"rank {rank}: PeerFailedError on the failing rank"
    wk.close()


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    comm = Comm(share_unique_id(rank), world, rank)
    exchanges = sys.argv[1:] or ["p2p", "p2p-exact", "nccl"]
    for exchange in exchanges:
        for case in CASES:
            run_case(case, exchange, comm, rank, world, dev)
        if world == 2:
            run_records_case(exchange, comm, rank, world, dev)
        run_pipelined_case(exchange, comm, rank, world, dev)
        if exchange in ("p2p", "p2p-exact"):
            run_failure_case(exchange, comm, rank, world, dev)
    comm.close()
    dist.barrier(device_ids=[local])
    if rank == 0:
        print(f"MGPU OK world={world} cases={len(CASES)} exchanges={exchanges}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
