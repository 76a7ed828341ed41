"""Per-round records of the GPU engine vs the reference's own metrics.csv.

tests/golden/metrics_n1.csv was written by the unmodified reference (its lock-step engine,
_make_record and the CLI's write_metrics_csv; tests/golden/make_metrics_golden.py). The same
run through CDSGDWorker + records.Recorder must give the same iter / epoch / loss / bytes /
compressed / wall_micros columns exactly and the same grad_norm to 1e-12 relative (the
reference takes np.linalg.norm of the fp64 round mean; the engine sums squares on the GPU)."""

import os

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("weights", ["f64", "f32"])
def test_records_match_reference_metrics_csv(tmp_path, weights):
    from paper_2106_10796_b200 import _lib
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import Layout
    from paper_2106_10796_b200.records import Recorder, read_metrics_csv, write_metrics_csv
    from paper_2106_10796_b200.worker import CDSGDWorker

    _lib.load()
    sizes, seed, k, warm, iters = [1000, 37, 16, 1], 0, 4, 2, 14
    layout = Layout.from_lengths(sizes)
    n = layout.total
    hp = HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=k, alpha=0.5, warmup_n=warm)
    wk = CDSGDWorker(layout, hp, O.synthetic_weights(seed, n), weights=weights)
    rec = Recorder(wk, batches_per_epoch=1)
    for t in range(iters):
        wk.step(torch.from_numpy(O.synthetic_grad(seed, t, 0, n)).cuda())
        rec.record(0.0)
    wk.flush()
    ours = rec.records()
    assert len(ours) == iters
    write_metrics_csv(tmp_path / "metrics.csv", ours)
    gold = read_metrics_csv(os.path.join(GOLD, "metrics_n1.csv"))
    mine = read_metrics_csv(tmp_path / "metrics.csv")
    for g, m in zip(gold, mine):
        assert (g.iteration, g.epoch, g.train_loss, g.bytes_pushed, g.compressed, g.wall_micros) == \
               (m.iteration, m.epoch, m.train_loss, m.bytes_pushed, m.compressed, m.wall_micros)
        assert abs(g.grad_norm - m.grad_norm) <= 1e-12 * g.grad_norm, (g, m)
