"""Golden vectors of the fp32-RESIDUAL FAST MODE (oracle/cdsgd_oracle.py quantize_f32).

The reference has no fp32 path (it computes in fp64, codec.py:176): the fast mode is pinned
to its own restatement of codec.py:181-193 in float32, whose outputs are frozen here so the
GPU kernel (cdsgd_quantize_f32r) and the restatement can both be checked against fixed
vectors. The one point where the two modes must agree is also recorded: from a ZERO
residual, fp32 and fp64 quantization give the same codes and the same residual (every
r' = g - e is exact in fp32), checked against the reference's own goldens
(codec_golden.npz) in tests/test_oracle_f32.py.

    python tests/golden/make_f32_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import cdsgd_oracle as O  # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(4321)
    cases = []
    for n in (1, 15, 16, 17, 100, 1000, 4099):
        cases.append((f"rand{n}", (0.4 * rng.standard_normal(n)).astype(np.float32),
                      (0.5 * rng.standard_normal(n)).astype(np.float32), 0.5))
    cases.append(("alpha0.3", (0.2 * rng.standard_normal(777)).astype(np.float32),
                  (0.3 * rng.standard_normal(777)).astype(np.float32), 0.3))
    sub = np.float32(1e-45)
    special_r = np.array([0.0, 0.0, 0.3, -0.2, 0.0, 0.0, -0.0, 0.0, 0.25, -0.25, 1e-38, -1e-38, 0.0, 0.0, 0.5, -0.5,
                          0.0, sub, -sub], dtype=np.float32)
    special_g = np.array([0.7, 0.0, 0.1, -0.4, 0.5, -0.5, -0.0, 1.7, 0.25, -0.25, 0.0, 0.0, -1.7, 3.0, 0.0, 0.0, sub,
                          0.0, -0.0], dtype=np.float32)
    cases.append(("special", special_r, special_g, 0.5))
    names = []
    for name, r, g, alpha in cases:
        w, rn = O.quantize_f32(r, g, alpha)
        out[f"q_{name}_r"], out[f"q_{name}_g"], out[f"q_{name}_alpha"] = r, g, np.float64(alpha)
        out[f"q_{name}_words"], out[f"q_{name}_rnew"] = w, rn
        names.append(name)
    out["q_names"] = np.array(names)
    # a 60-step stream with the residual carried (fp32)
    rs = np.zeros(300, np.float32)
    sg, sw, sr = [], [], []
    for t in range(60):
        g = O.synthetic_grad(7, t, 0, 300)
        w, rs = O.quantize_f32(rs, g, 0.5)
        sg.append(g)
        sw.append(w)
        sr.append(rs.copy())
    out["stream_g"], out["stream_words"], out["stream_r"] = np.stack(sg), np.stack(sw), np.stack(sr)
    # non-finite: first index, residual untouched
    g = np.concatenate([np.zeros(40, np.float32), [np.nan], np.zeros(5, np.float32), [np.inf]]).astype(np.float32)
    try:
        O.quantize_f32(np.zeros(47, np.float32), g, 0.5)
        raise AssertionError("expected OracleNumericError")
    except O.OracleNumericError as exc:
        out["e_g"], out["e_index"] = g, np.int64(exc.index)
    np.savez_compressed(os.path.join(HERE, "codec_f32_golden.npz"), **out)
    print("wrote codec_f32_golden.npz:", len(names), "cases")


if __name__ == "__main__":
    main()
