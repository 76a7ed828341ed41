"""BASELINE.json configs[0] — the reference's own CPU-runnable case — end to end on the GPU.

Config (i): CD-SGD, threshold 0.5, k = 4, warm-up 5, a
1M-element synthetic fp32 gradient, 100 steps, 2 workers; plus the 2-key [1048575, 1]
variant (a key whose length is not a multiple of 16 and a 1-element key). Parity contract
(BASELINE.md §2): residuals bitwise every round, global and compute weights within
rtol 1e-5 / atol 1e-6 every round, against the C restatement of the reference round
(oracle/cdsgd_oracle.c, pinned bitwise to the reference's golden traces by
tests/test_oracle_cport.py / test_oracle_golden.py).

* N = 2 simulated on one GPU through the C ABI (tests/localsim.py): the fused round F,
  K1, K2 and K3 with the local update, one W replica per worker (replicas bitwise equal).
* N = 1 through the public API (CDSGDWorker -> cdsgd_engine).
* alpha = 0.3 at N = 8 (and N = 3): partial sums j*alpha are not all representable, so
  F and K2 must decode with the reference's sequential ascending-worker fp64 sum
  (engine.py:249-255) instead of the count table; W is checked BITWISE against a fp32
  mirror of that arithmetic (W -= (float)(eta * mean)) every round.
"""

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O
from oracle import cpu_port

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.fixture(scope="module")
def pkg():
    from paper_2106_10796_b200 import _lib, engine, layout, worker

    _lib.load()
    torch.cuda.set_device(0)
    if cpu_port.load() is None:
        pytest.skip("C port not built (make -C oracle)")
    return engine, layout, worker


def grads_of(seed, t, N, n):
    return np.stack([O.synthetic_grad(seed, t, w, n) for w in range(N)])


@pytest.mark.parametrize("weights", ["f64", "f32"])
@pytest.mark.parametrize("sizes", [[1_048_576], [1_048_575, 1]], ids=["1M", "1048575+1"])
def test_config_i_two_workers_local_sim_100_rounds(pkg, sizes, weights):
    from localsim import LocalSim

    _, L, _ = pkg
    layout = L.Layout.from_lengths(sizes)
    n, N, T = layout.total, 2, 100
    w0 = O.synthetic_weights(0, n)
    sim = LocalSim(layout, N, w0, k=4, alpha=0.5, eta_g=0.1, eta_l=0.4, warmup=5, weights=weights)
    port = cpu_port.CPortEngine(w0.astype(np.float64), sizes, N, k=4, alpha=0.5, eta_g=0.1, eta_l=0.4, warmup=5)
    seen = set()
    for t in range(T):
        for w in range(N):  # compute weights of round t (engine.py:335-343)
            ref = port.loc[w] if t >= max(port.warm, 1) else port.W
            np.testing.assert_allclose(sim.compute_weights(w).cpu().numpy(), ref, rtol=RTOL, atol=ATOL,
                                       err_msg=f"compute weights round {t} worker {w}")
        g = grads_of(0, t, N, n)
        sim.step([torch.from_numpy(g[w]).cuda() for w in range(N)])
        port.step(g)
        seen.update(sim.kernels[-1])
        assert sim.compressed(t) == port.compressed(t)
        for w in range(N):
            assert np.array_equal(bits(sim.residual(w).cpu().numpy()), bits(port.res[w])), f"residual t={t} w={w}"
            if port.compressed(t):
                assert np.array_equal(sim.words(t, w).cpu().numpy(), port.words[w]), f"codes t={t} w={w}"
        assert torch.equal(sim.W[0], sim.W[1]), f"W replicas differ after round {t}"
    sim.flush()
    for w in range(N):
        np.testing.assert_allclose(sim.W[w].cpu().numpy(), port.W, rtol=RTOL, atol=ATOL)
    if weights == "f64":  # fp64 W: only the fp32 correction sums (the all-reduce) differ from the reference
        np.testing.assert_allclose(sim.W[0].cpu().numpy(), port.W, rtol=0, atol=1e-7)
    assert sim.errors() == [[-1, -1]] * N
    # every kernel of the engine's choreography ran
    assert {"F", "F_L", "K1", "K2", "K3"} <= seen or {"F", "K2", "K3"} <= seen, seen


@pytest.mark.parametrize("weights", ["f64", "f32"])
@pytest.mark.parametrize("sizes", [[1_048_576], [1_048_575, 1]], ids=["1M", "1048575+1"])
def test_config_i_worker_api_100_rounds(pkg, sizes, weights):
    """N = 1 through the public API. fp64 weights (exact mode) are the reference's W BIT FOR BIT
    every round (every update is the reference's own fp64 operation and, at N = 1, the
    correction mean is g itself), and the compute weights are the reference's rounded once
    to fp32; fp32 weights stay within the contract tolerance."""
    E, L, Wk = pkg
    layout = L.Layout.from_lengths(sizes)
    n, T = layout.total, 100
    w0 = O.synthetic_weights(1, n)
    hp = E.HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5, warmup_n=5)
    wk = Wk.CDSGDWorker(layout, hp, w0, weights=weights)
    port = cpu_port.CPortEngine(w0.astype(np.float64), sizes, 1, k=4, alpha=0.5, eta_g=0.1, eta_l=0.4, warmup=5)
    for t in range(T):
        ref = port.loc[0] if t >= max(port.warm, 1) else port.W
        np.testing.assert_allclose(wk.compute_weights().cpu().numpy(), ref, rtol=RTOL, atol=ATOL,
                                   err_msg=f"compute weights round {t}")
        g = grads_of(1, t, 1, n)
        wk.step(torch.from_numpy(g[0]).cuda())
        port.step(g)
        assert wk.round_compressed(t) == port.compressed(t)
        assert np.array_equal(bits(wk.residual.cpu().numpy()), bits(port.res[0])), f"residual round {t}"
        if weights == "f64" and t >= port.warm:
            cw = wk.compute_weights().cpu().numpy()
            assert np.array_equal(cw.view(np.uint32), port.loc[0].astype(np.float32).view(np.uint32)), \
                f"compute weights != fl32(reference) round {t}"
    wk.flush()
    np.testing.assert_allclose(wk.weights.cpu().numpy(), port.W, rtol=RTOL, atol=ATOL)
    if weights == "f64":
        assert np.array_equal(bits(wk.weights.cpu().numpy()), bits(port.W)), "fp64 W not bitwise the reference's"


@pytest.mark.parametrize("weights", ["f32", "f64"])
@pytest.mark.parametrize("N,alpha", [(8, 0.3), (3, 0.3), (8, 0.5), (4, 0.1)])
def test_non_dyadic_alpha_decode_bitwise(pkg, N, alpha, weights):
    """All rounds compressed (k large, no warm-up): every apply is F (or K2 for the last);
    W must equal, bit for bit, fp32 W minus (float)(eta * mean) with mean the reference's
    ascending fp64 sum of decoded codes / N — whether or not alpha's multiples are exact."""
    from localsim import LocalSim

    _, L, _ = pkg
    sizes = [4099, 512, 77, 3000]
    layout = L.Layout.from_lengths(sizes)
    n, T, eta = layout.total, 12, 0.1
    w0 = O.synthetic_weights(7, n)
    sim = LocalSim(layout, N, w0, k=10_000, alpha=alpha, eta_g=eta, eta_l=0.4, warmup=0, weights=weights)
    port = cpu_port.CPortEngine(w0.astype(np.float64), sizes, N, k=10_000, alpha=alpha, eta_g=eta, eta_l=0.4)
    Wm = w0.astype(np.float32).copy()  # fp32 mirror of the apply
    prev_mean = None
    Wref_prev = None
    for t in range(T):
        g = grads_of(7, t, N, n)
        sim.step([torch.from_numpy(g[w]).cuda() for w in range(N)])
        port.step(g)
        if t >= 1:  # round t-1 was applied inside this step (F)
            assert sim.kernels[-1] == ["F"], sim.kernels[-1]
            got = sim.W[0].cpu().numpy()
            if weights == "f32":
                assert np.array_equal(got.view(np.uint32), Wm.view(np.uint32)), f"W not bitwise after round {t - 1}"
            else:  # fp64: the reference's W itself (the C port applied rounds 0..t)
                assert np.array_equal(bits(got), bits(Wref_prev)), f"W not bitwise after round {t - 1}"
            gsq = float(prev_mean @ prev_mean)
            assert abs(sim.gnorm.item() - gsq) <= 1e-12 * max(gsq, 1.0), (sim.gnorm.item(), gsq)
        for w in range(N):
            assert np.array_equal(bits(sim.residual(w).cpu().numpy()), bits(port.res[w])), f"residual t={t} w={w}"
        mean = O.server_aggregate([O.dequantize_layout(port.words[w], alpha, sizes) for w in range(N)])
        Wm = (Wm - (eta * mean).astype(np.float32)).astype(np.float32)
        prev_mean = mean
        Wref_prev = port.W.copy()
        for w in range(1, N):
            assert torch.equal(sim.W[0], sim.W[w])
    sim.flush()  # K2 applies the last round
    if weights == "f32":
        assert np.array_equal(sim.W[0].cpu().numpy().view(np.uint32), Wm.view(np.uint32))
    else:
        assert np.array_equal(bits(sim.W[0].cpu().numpy()), bits(port.W))
    np.testing.assert_allclose(sim.W[0].cpu().numpy(), port.W, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("weights", ["f32", "f64"])
def test_weight_drift_envelope(pkg, weights):
    """W and loc are fp32 on the GPU (the reference keeps fp64, SPEC 'Use 64-bit reals
    internally'): each round rounds W once to fp32. Over a long horizon (2,000 rounds of the
    ResNet-20 layout, k = 4, warm-up 5, N = 1) the deviation from the fp64 reference (C
    port) must stay inside rtol 1e-5 + atol 1e-6 up to 100 rounds and inside the random-walk
    envelope rtol 1e-5 + max(1e-6 sqrt(T/100), 2^-24 max|W| sqrt(T)) beyond;
    the measured curve is printed and written to gpurun_out/drift_envelope.json (DESIGN.md §3
    quotes it)."""
    import json
    import os

    E, L, Wk = pkg
    layout = L.by_name("resnet20")
    sizes = layout.lengths
    n, T = layout.total, 2000
    w0 = O.synthetic_weights(3, n)
    hp = E.HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5, warmup_n=5)
    wk = Wk.CDSGDWorker(layout, hp, w0, weights=weights)
    port = cpu_port.CPortEngine(w0.astype(np.float64), sizes, 1, k=4, alpha=0.5, eta_g=0.1, eta_l=0.4, warmup=5)
    curve = []
    for t in range(T):
        g = grads_of(3, t, 1, n)
        wk.step(torch.from_numpy(g[0]).cuda())
        port.step(g)
        if (t + 1) % 100 == 0:
            assert np.array_equal(bits(wk.residual.cpu().numpy()), bits(port.res[0])), f"residual round {t}"
            wk.flush()
            W = wk.weights.cpu().numpy().astype(np.float64)
            loc = wk.compute_weights().cpu().numpy().astype(np.float64)
            dW, dl = np.abs(W - port.W), np.abs(loc - port.loc[0])
            curve.append({"round": t + 1,
                          "max_abs_W": float(dW.max()), "max_rel_W": float((dW / np.maximum(np.abs(port.W), 1e-30)).max()),
                          "excess_W": float((dW - RTOL * np.abs(port.W)).max()),
                          "max_abs_loc": float(dl.max()), "excess_loc": float((dl - RTOL * np.abs(port.loc[0])).max()),
                          "max_abs_Wref": float(np.abs(port.W).max())})
            # the contract tolerance (rtol 1e-5, atol 1e-6) up to the BASELINE horizon of 100 rounds;
            # beyond it the absolute part grows like a random walk of one fp32 rounding (<= half
            # an ulp of the largest |W|) per round: atol(T) = max(1e-6 sqrt(T/100), 2^-24 max|W| sqrt(T))
            T1 = t + 1
            atol_t = ATOL if T1 <= 100 else max(ATOL * (T1 / 100) ** 0.5,
                                                2.0 ** -24 * float(np.abs(port.W).max()) * T1 ** 0.5)
            curve[-1]["envelope_atol"] = atol_t
            if weights == "f64":  # exact mode: no drift at all
                assert np.array_equal(bits(wk.weights.cpu().numpy()), bits(port.W)), f"W after {t + 1} rounds"
            np.testing.assert_allclose(W, port.W, rtol=RTOL, atol=atol_t, err_msg=f"W after {t + 1} rounds")
            np.testing.assert_allclose(loc, port.loc[0], rtol=RTOL, atol=atol_t, err_msg=f"loc after {t + 1} rounds")
    out = {"weights": weights, "layout": "resnet20", "n": n, "rounds": T, "k": 4, "warmup_n": 5, "alpha": 0.5, "eta_g": 0.1,
           "eta_l": 0.4, "tolerance": {"rtol": RTOL, "atol": ATOL}, "curve": curve}
    print(json.dumps(out["curve"][-1]))
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, f"drift_envelope_{weights}.json"), "w") as f:
            json.dump(out, f, indent=1)


@pytest.mark.parametrize("N", [4, 8])
def test_half_tile_fused_round_many_ranks_bitwise(pkg, N):
    """Layouts above the small-layout threshold with several ranks' codes and fp64 W run the
    fused round on HALF tiles (no register spill; for N > 5 also with per-word count sums):
    W bitwise against the reference's fp64 W (C port) and residuals bitwise, every round."""
    from localsim import LocalSim

    _, L, _ = pkg
    sizes = [2_600_000, 77, 3000]  # > 4,736 tiles: whole-/half-tile tasks, not chunk tasks
    layout = L.Layout.from_lengths(sizes)
    n, T, eta = layout.total, 4, 0.1
    w0 = O.synthetic_weights(11, n)
    sim = LocalSim(layout, N, w0, k=10_000, alpha=0.5, eta_g=eta, eta_l=0.4, warmup=0, weights="f64")
    port = cpu_port.CPortEngine(w0.astype(np.float64), sizes, N, k=10_000, alpha=0.5, eta_g=eta, eta_l=0.4)
    Wref_prev = None
    for t in range(T):
        g = grads_of(11, t, N, n)
        sim.step([torch.from_numpy(g[w]).cuda() for w in range(N)])
        port.step(g)
        if t >= 1:
            assert sim.kernels[-1] == ["F"], sim.kernels[-1]
            assert np.array_equal(bits(sim.W[0].cpu().numpy()), bits(Wref_prev)), f"W not bitwise after round {t - 1}"
        for w in range(N):
            assert np.array_equal(bits(sim.residual(w).cpu().numpy()), bits(port.res[w])), f"residual t={t} w={w}"
        Wref_prev = port.W.copy()
    sim.flush()
    assert np.array_equal(bits(sim.W[0].cpu().numpy()), bits(port.W))
