"""The C restatement (CPU baseline) is bit-identical to the NumPy oracle and to the
reference golden traces, for any OpenMP thread count."""

import numpy as np
import pytest

from oracle import cdsgd_oracle as O
from oracle import cpu_port


@pytest.fixture(scope="module")
def lib():
    lib = cpu_port.load()
    if lib is None:
        pytest.skip("C port not built (make -C oracle)")
    return lib


def test_cport_quantize_layout_bitwise(lib):
    rng = np.random.default_rng(0)
    for sizes in ([1], [15, 16, 17], [1048575, 1], [3, 1000, 5, 513]):
        n = sum(sizes)
        r = rng.standard_normal(n) * 0.4
        g = (rng.standard_normal(n) * 0.6).astype(np.float32)
        ow, orn = O.quantize_layout(r, g, 0.5, sizes)
        for th in (1, 3):
            lib.cdsgd_ref_set_threads(th)
            rr = r.copy()
            words = np.zeros(ow.shape[0], np.uint32)
            sz = np.asarray(sizes, np.int64)
            bad = lib.cdsgd_ref_quantize_layout(cpu_port._p(rr), cpu_port._p(g), cpu_port._p(rr), cpu_port._p(words),
                                                cpu_port._p(sz), len(sizes), 0.5)
            assert bad == -1
            assert np.array_equal(words, ow) and np.array_equal(rr.view(np.uint64), orn.view(np.uint64))
    g = np.zeros(40, np.float32)
    g[33] = np.nan
    r = np.zeros(40)
    sz = np.asarray([30, 10], np.int64)
    assert lib.cdsgd_ref_quantize_layout(cpu_port._p(r), cpu_port._p(g), cpu_port._p(r),
                                         cpu_port._p(np.zeros(3, np.uint32)), cpu_port._p(sz), 2, 0.5) == 33


def test_cport_engine_matches_golden(lib, engine_golden):
    E = engine_golden
    for name in ("cd_n2_k4_w5", "cd_n1_k3_w0", "cd_n4_k2_w1", "cd_n8_k4_w5", "cd_n3_k4_w3", "cd_n2_a03"):
        p = f"{name}_"
        nwk, k, warm, iters, *_ = (int(x) for x in E[p + "cfg"])
        eta_g, eta_l, alpha = (float(x) for x in E[p + "hyper"])
        eng = cpu_port.CPortEngine(E[p + "w0"], E[p + "sizes"], nwk, k=k, alpha=alpha, eta_g=eta_g, eta_l=eta_l,
                                   warmup=warm)
        for t in range(iters):
            eng.step(E[p + "grads"][t])
            assert np.array_equal(eng.W.view(np.uint64), E[p + "weights_after"][t].view(np.uint64)), (name, t)
            if t + 1 < iters and t + 1 >= max(warm, 1):
                for w in range(nwk):
                    assert np.array_equal(eng.loc[w], E[p + "compute"][t + 1, w]), (name, t, w)
        for w in range(nwk):
            assert np.array_equal(eng.res[w], E[p + "final_residual"][w]), (name, w)


def test_time_rounds_smoke(lib):
    secs, kind, cores, impl = cpu_port.time_rounds([1000, 24], 2, 4, 0.5, 4)
    assert secs > 0 and kind == "port" and cores >= 1
