"""World-size-2 CPU (gloo) tests of the N>1 host-side logic.

* NCCL bootstrap: rank 0's ncclUniqueId (from libcdsgd_b200.so) reaches every rank
  intact through torch.distributed (comm.share_unique_id).
* Replicated parameter server: each rank quantizes only its own gradient, the packed
  words are all-gathered, and every rank decodes/sums in ascending rank order and
  applies the update to its own W replica — the design of the NCCL engine. On CPU
  the arithmetic is done by the oracle (test infrastructure) and the exchange by gloo;
  the result must equal the reference's lock-step parameter server bitwise
  (engine.py:249-255, 509-511) and replicas must agree bitwise.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _uid_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    from paper_2106_10796_b200 import comm

    uid = comm.share_unique_id(rank)
    q.put((rank, uid))
    dist.destroy_process_group()


def _replica_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    from oracle import cdsgd_oracle as O

    sizes = [1000, 37, 16, 1]
    n = sum(sizes)
    hp = O.OracleHP("cdsgd", world, 0.1, 0.4, 4, 0.5, 3)
    w0 = O.synthetic_weights(9, n).astype(np.float64)
    ref = O.LockstepOracle(w0, sizes, hp)          # every rank also runs the full PS for comparison
    W = w0.copy()                                   # this rank's replica
    res = np.zeros(n)
    nw = sum((s + 15) // 16 for s in sizes)
    ok = True
    for t in range(14):
        grads = [O.synthetic_grad(9, t, w, n) for w in range(world)]
        comp = ref._push_compressed(ref.workers[0])
        if comp:
            words, res = O.quantize_layout(res, grads[rank], hp.alpha, sizes)
            gathered = [torch.zeros(nw, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(words.astype(np.int64)))
            deq = [O.dequantize_layout(g.numpy().astype(np.uint32), hp.alpha, sizes) for g in gathered]
        else:
            gathered = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(grads[rank].astype(np.float64)))
            deq = [g.numpy() for g in gathered]
        W -= hp.eta_global * O.server_aggregate(deq)
        ref.step(grads)
        ok &= bool(np.array_equal(W, ref.W)) and bool(np.array_equal(res, ref.workers[rank].residual))
    allW = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allW, torch.from_numpy(W))
    ok &= all(torch.equal(allW[0], a) for a in allW)
    q.put((rank, ok))
    dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_nccl_unique_id_broadcast_gloo():
    out = _run(_uid_worker)
    assert len(out[0]) == 128 and out[0] == out[1]


def test_replicated_server_matches_lockstep_gloo():
    out = _run(_replica_worker)
    assert out[0] and out[1]
