"""Golden metrics.csv from the UNMODIFIED reference (cdsgd 0.1.0) — build container only.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_metrics_golden.py

Runs the reference's lock-step engine (Worker / ServerNode / _run_lockstep, engine.py:288-663)
on synthetic gradients (``engine.loss_and_grad`` replaced, SURVEY §8c recipe: loss 0.0),
turns every round into an IterationRecord with the reference's own ``_make_record``
(engine.py:593-611) and writes it with the reference CLI's ``write_metrics_csv``
(cli.py:39-56). tests/test_gpu_records.py reproduces the same run on the GPU engine and
compares the files column by column.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import cdsgd.cli as cli  # noqa: E402
import cdsgd.engine as engine  # noqa: E402
from cdsgd.numcore import Dataset, KeyedVector, Layout, ModelSpec  # noqa: E402

CASES = {
    # name: (sizes, n_workers, k, warmup, iters, seed)
    "metrics_n1": ([1000, 37, 16, 1], 1, 4, 2, 14, 0),
    "metrics_n2": ([640, 7, 33], 2, 3, 1, 11, 4),
}


def synthetic_grad(seed, t, w, n, scale=0.3):
    return (scale * np.random.default_rng([seed, t, w]).standard_normal(n)).astype(np.float32)


def synthetic_weights(seed, n):
    return np.random.default_rng([seed, 999]).standard_normal(n).astype(np.float32)


def run(name, sizes, n_workers, k, warmup, iters, seed):
    layout = Layout([(f"k{i}", s) for i, s in enumerate(sizes)])
    n = layout.total
    calls = {"c": 0}

    def fake_loss_and_grad(model, weights, X, y):
        t, w = divmod(calls["c"], n_workers)
        calls["c"] += 1
        return 0.0, KeyedVector(synthetic_grad(seed, t, w, n).astype(np.float64), layout)

    saved = engine.loss_and_grad
    engine.loss_and_grad = fake_loss_and_grad
    try:
        hp = engine.HyperParams(algo="cdsgd", workers=n_workers, eta_global=0.1, eta_local=0.4, k=k, alpha=0.5,
                                warmup_n=warmup, batch_size=1, iters=iters, seed=seed).validate()
        init = KeyedVector(synthetic_weights(seed, n).astype(np.float64), layout)
        server = engine.ServerNode(init, hp)
        ds = Dataset(np.zeros((n_workers, 1)), np.zeros(n_workers)).with_shards(n_workers)
        workers = [engine.Worker(w, ModelSpec("linear-regression", 1, 1), ds, hp, init, np.random.default_rng(w))
                   for w in range(n_workers)]
        rounds = engine._run_lockstep(server, workers, iters, layout)
        records = [engine._make_record(t, rounds[t], server, 0) for t in range(iters)]
    finally:
        engine.loss_and_grad = saved
    cli.write_metrics_csv(os.path.join(HERE, f"{name}.csv"), records)


def main():
    for name, case in CASES.items():
        run(name, *case)
        print("wrote", name)


if __name__ == "__main__":
    main()
