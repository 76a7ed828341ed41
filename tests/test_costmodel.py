"""The time model (paper Eq. 6-9) against the reference's own outputs (tests/golden/
costmodel_golden.npz, written by importing cdsgd.costmodel), plus its error behaviour.
Host-only; the B200 calibration that feeds it is scripts/calibrate_costmodel.py."""

import os
import warnings

import numpy as np
import pytest

from paper_2106_10796_b200 import costmodel as cm

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "costmodel_golden.npz"))


def _params(row):
    tau, phi, psi, delta, k = row
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return cm.CostParams(tau=tau, phi=phi, psi=psi, delta=delta, k=int(k))


def test_golden_grid_exact():
    for j, row in enumerate(G["cm_params"]):
        p = _params(row)
        assert (cm.t_ssgd(p), cm.t_loc(p), cm.t_bit(p), cm.avg_cd(p)) == tuple(G["cm_avg"][j]), row
        got = [(cm.comm_cd(i, p), cm.t_cd(i, p), cm.saving_vs_loc(i, p), cm.saving_vs_bit(i, p))
               for i in range(1, 11)]
        assert np.array_equal(np.array(got), G["cm_per_i"][j]), row
        assert cm.classify_regime(p) == str(G["cm_regime"][j]), row
        assert [r[3] for r in cm.timeline(p, 10)] == list(G["cm_timeline_cum"][j]), row


def test_grid_covers_every_regime_and_negative_saving():
    assert set(G["cm_regime"]) == {cm.REGIME_COMPUTE, cm.REGIME_MIXED, cm.REGIME_COMM}
    assert (G["cm_per_i"][:, :, 3] < 0).any()  # Eq. 8 case 3: correction slower than BIT-SGD


def test_errors_and_warning():
    with pytest.raises(ValueError):
        cm.CostParams(tau=-1, phi=1, psi=0.5, delta=0, k=4)
    with pytest.raises(ValueError):
        cm.CostParams(tau=1, phi=1, psi=0.5, delta=0, k=0)
    with pytest.warns(UserWarning):
        cm.CostParams(tau=1, phi=1, psi=2, delta=0, k=4)
    p = cm.CostParams(tau=1, phi=2, psi=0.5, delta=0.1, k=4)
    with pytest.raises(ValueError):
        cm.comm_cd(0, p)
    with pytest.raises(ValueError):
        cm.timeline(p, 0)
    # comm-bound average = ((k-1)(delta+psi) + phi) / k (PAPER eq. after 8)
    q = cm.CostParams(tau=0.1, phi=2, psi=0.5, delta=0.1, k=4)
    assert cm.avg_cd(q) == pytest.approx((3 * 0.6 + 2) / 4)


@pytest.mark.gpu
def test_calibration_runs_on_one_gpu():
    """The B200 calibration path (scripts/calibrate_costmodel.py) end to end at N=1 on a
    small model: measured constants are positive and every algorithm trains."""
    import sys

    import torch

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "scripts"))
    import calibrate_costmodel as cal

    from paper_2106_10796_b200 import _lib

    _lib.load()
    out = cal.calibrate(["tiny"], 1, 0, None, torch.device("cuda", 0))["models"]["tiny"]
    assert all(v > 0 for k, v in out["constants_s"].items() if k != "psi")
    assert set(out["measured_iter_s"]) == set(cm.ALGOS)
    assert out["regime"] in (cm.REGIME_COMPUTE, cm.REGIME_MIXED, cm.REGIME_COMM)
