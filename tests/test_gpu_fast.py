"""fp32-residual FAST MODE on the GPU (opt-in; SURVEY §8(b) cdsgd_quantize_seg_f32r, §8(c)
fp32 restatement oracle): bit-exact against the fp32 restatement of codec.py:181-193
(oracle quantize_f32) and its frozen goldens; the engine in fast mode (fp32 residual +
fp32 weights) against the lock-step oracle with the fp32 quantizer, residual bitwise every
round, weights within the contract tolerance."""

import os

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RTOL, ATOL = 1e-5, 1e-6


@pytest.fixture(scope="module")
def lib():
    from paper_2106_10796_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)
    return _lib


def q32(_lib, sizes, r, g, alpha):
    """cdsgd_quantize_f32r over a layout; returns (words, r_out, err)."""
    from paper_2106_10796_b200.layout import Layout

    lay = Layout.from_lengths(sizes)
    rd = torch.from_numpy(np.ascontiguousarray(r, np.float32)).cuda()
    gd = torch.from_numpy(np.ascontiguousarray(g, np.float32)).cuda()
    ro = torch.empty_like(rd)
    words = torch.zeros(max(lay.n_words, 1), dtype=torch.int32, device="cuda")
    err = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().cdsgd_quantize_f32r(lay.handle().ptr, gd.data_ptr(), rd.data_ptr(), ro.data_ptr(),
                                              words.data_ptr(), alpha, err.data_ptr(), 0,
                                              torch.cuda.current_stream().cuda_stream), "quantize_f32r")
    return words.cpu().numpy().view(np.uint32)[:lay.n_words], ro.cpu().numpy(), int(err[0].item())


def test_f32r_goldens(lib):
    f = np.load(os.path.join(GOLD, "codec_f32_golden.npz"))
    for name in f["q_names"]:
        r, g = f[f"q_{name}_r"], f[f"q_{name}_g"]
        w, ro, e = q32(lib, [len(r)], r, g, float(f[f"q_{name}_alpha"]))
        assert e == -1, name
        assert np.array_equal(w, f[f"q_{name}_words"]), name
        assert np.array_equal(ro.view(np.uint32), f[f"q_{name}_rnew"].view(np.uint32)), name
    r = np.zeros(300, np.float32)
    for t in range(60):
        w, r, _ = q32(lib, [300], r, f["stream_g"][t], 0.5)
        assert np.array_equal(w, f["stream_words"][t]) and np.array_equal(r, f["stream_r"][t]), t
    w, ro, e = q32(lib, [47], np.zeros(47, np.float32), f["e_g"], 0.5)
    assert e != -1 and (e & ((1 << 40) - 1)) == int(f["e_index"])


@pytest.mark.parametrize("sizes", [[1], [17, 4099], [1 << 20], [1048575, 1], [5000, 33, 1024, 3]])
def test_f32r_vs_oracle(lib, sizes):
    n = sum(sizes)
    rng = np.random.default_rng(n)
    r = (0.4 * rng.standard_normal(n)).astype(np.float32)
    for t in range(3):
        g = (0.5 * rng.standard_normal(n)).astype(np.float32)
        w, ro, e = q32(lib, sizes, r, g, 0.5)
        ow, orr = O.quantize_layout_f32(r, g, 0.5, sizes)
        assert e == -1
        assert np.array_equal(w, ow) and np.array_equal(ro.view(np.uint32), orr.view(np.uint32)), t
        r = ro


@pytest.mark.parametrize("case", [([3_000_000, 4099, 17], 4, 1, 9), ([1000, 37, 16, 1], 4, 5, 16), ([700], 2, 0, 10)])
def test_engine_fast_mode_vs_oracle(lib, case):
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import Layout
    from paper_2106_10796_b200.worker import CDSGDWorker

    sizes, k, warm, iters = case
    layout = Layout.from_lengths(sizes)
    n = layout.total
    hp = HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=k, alpha=0.5, warmup_n=warm)
    w0 = O.synthetic_weights(2, n)
    wk = CDSGDWorker(layout, hp, w0, weights="f32", residual="f32")
    assert wk.residual.dtype == torch.float32
    orc = O.LockstepOracle(w0.astype(np.float64), sizes, O.OracleHP("cdsgd", 1, 0.1, 0.4, k, 0.5, warm),
                           residual="f32")
    for t in range(iters):
        np.testing.assert_allclose(wk.compute_weights().cpu().numpy(), orc.compute_weights(0), rtol=RTOL, atol=ATOL,
                                   err_msg=f"compute weights round {t}")
        g = O.synthetic_grad(2, t, 0, n)
        wk.step(torch.from_numpy(g).cuda())
        orc.step([g])
        assert np.array_equal(wk.residual.cpu().numpy().view(np.uint32), orc.workers[0].residual.view(np.uint32)), t
    wk.flush()
    np.testing.assert_allclose(wk.weights.cpu().numpy(), orc.W, rtol=RTOL, atol=ATOL)


def test_fast_mode_needs_fp32_weights(lib):
    from paper_2106_10796_b200.engine import ConfigError, HyperParams
    from paper_2106_10796_b200.layout import Layout
    from paper_2106_10796_b200.worker import CDSGDWorker

    with pytest.raises(ConfigError):
        CDSGDWorker(Layout.from_lengths([64]), HyperParams(algo="cdsgd", workers=1), np.zeros(64, np.float32),
                    residual="f32")
