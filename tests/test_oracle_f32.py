"""The fp32-residual fast-mode oracle (quantize_f32, a float32 restatement of
codec.py:181-193) against its frozen goldens, and its one anchor to the reference: from a
zero residual every r' = g - e is exact in fp32, so the first step equals the reference's
fp64 step bit for bit (codes) and value for value (residual) — checked against the
reference-generated stream in codec_golden.npz."""

import os

import numpy as np
import pytest

from oracle import cdsgd_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def f32g():
    return np.load(os.path.join(GOLD, "codec_f32_golden.npz"))


def test_quantize_f32_matches_goldens(f32g):
    for name in f32g["q_names"]:
        w, r = O.quantize_f32(f32g[f"q_{name}_r"], f32g[f"q_{name}_g"], float(f32g[f"q_{name}_alpha"]))
        assert np.array_equal(w, f32g[f"q_{name}_words"]), name
        assert np.array_equal(r.view(np.uint32), f32g[f"q_{name}_rnew"].view(np.uint32)), name
    rs = np.zeros(300, np.float32)
    for t in range(60):
        w, rs = O.quantize_f32(rs, f32g["stream_g"][t], 0.5)
        assert np.array_equal(w, f32g["stream_words"][t]) and np.array_equal(rs, f32g["stream_r"][t]), t
    with pytest.raises(O.OracleNumericError) as ei:
        O.quantize_f32(np.zeros(47, np.float32), f32g["e_g"], 0.5)
    assert ei.value.index == int(f32g["e_index"]) == 40


def test_first_step_from_zero_equals_reference(codec_golden):
    g0 = codec_golden["stream_g"][0]
    w, r = O.quantize_f32(np.zeros_like(g0, dtype=np.float32), g0, 0.5)
    assert np.array_equal(w, codec_golden["stream_words"][0])
    assert np.array_equal(r.astype(np.float64), codec_golden["stream_r"][0])


def test_fast_mode_diverges_from_reference_later(codec_golden):
    """Documented, not a bug: carried fp32 residuals drift from the fp64 ones,
    which is why the fast mode is opt-in and pinned to its own restatement."""
    rs = np.zeros(300, np.float32)
    same_r = True
    for t in range(60):
        w, rs = O.quantize_f32(rs, codec_golden["stream_g"][t], 0.5)
        same_r &= np.array_equal(rs.astype(np.float64), codec_golden["stream_r"][t])
    assert not same_r
