"""GPU parity of the fused step (K1 + exchange + K2/K3 + local update).

* The native engine (N=1) against the lock-step oracle: residuals bit-exact every
  round, compute weights (W or loc) and final W within the fp32 tolerance
  rtol=1e-5, atol=1e-6, for every algorithm / warm-up / k.
* N simulated workers on one GPU ("local-sim", the analogue of the reference's
  lock-step scheduler): each worker's K1 writes its slot of one gathered buffer,
  K2/K3 apply on a shared W; checked against the reference's own golden engine
  traces (tests/golden/engine_golden.npz) for N in {2, 3, 4, 8}.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.fixture(scope="module")
def pkg():
    import paper_2106_10796_b200 as p
    from paper_2106_10796_b200 import _lib, engine, layout, worker

    _lib.load()
    torch.cuda.set_device(0)
    return p, engine, layout, worker


CASES = [
    # algo, sizes, k, warmup, iters, alpha, force, bypass
    # > 2 tiles per resident warp: the whole-tile (CH=4) path of the fused kernel
    ("cdsgd", [3_000_000, 4099, 17], 4, 1, 9, 0.5, False, False),
    # 1,500 keys (some misaligned, some < 1 tile): multi-round warp-collective key seeks and
    # long cursor jumps between dynamic claims, on the whole-tile path (> 2 tiles per warp)
    ("cdsgd", [((i * 7919) % 4000) + 1 for i in range(1500)], 4, 1, 9, 0.5, False, False),
    ("cdsgd", [1000, 37, 16, 1], 4, 5, 16, 0.5, False, False),
    ("cdsgd", [300], 3, 0, 12, 0.5, False, False),
    ("cdsgd", [4099, 512, 3], 2, 1, 11, 0.5, False, False),
    ("cdsgd", [700], 4, 2, 13, 0.5, False, False),
    ("cdsgd", [700], 1, 2, 7, 0.5, False, False),
    ("cdsgd", [513, 64], 4, 3, 10, 0.3, False, False),
    ("cdsgd", [150], 4, 2, 8, 0.5, True, False),
    ("cdsgd", [150], 4, 0, 8, 0.5, False, True),
    ("bitsgd", [100, 28], 5, 5, 6, 0.5, False, False),
    ("lusgd", [100, 28], 5, 2, 6, 0.5, False, False),
    ("ssgd", [77], 5, 5, 5, 0.5, False, False),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-k{c[2]}-w{c[3]}-{i}" for i, c in enumerate(CASES)])
def test_engine_n1_matches_oracle(pkg, case):
    _, E, L, Wk = pkg
    algo, sizes, k, warm, iters, alpha, force, bypass = case
    layout = L.Layout.from_lengths(sizes)
    n = layout.total
    hp = E.HyperParams(algo=algo, workers=1, eta_global=0.1, eta_local=0.4, k=k, alpha=alpha, warmup_n=warm)
    w0 = O.synthetic_weights(1, n)
    wk = Wk.CDSGDWorker(layout, hp, w0, force_compress=force, bypass_local=bypass)
    orc = O.LockstepOracle(w0.astype(np.float64), sizes,
                           O.OracleHP(algo, 1, 0.1, 0.4, k, alpha, warm, force, bypass))
    for t in range(iters):
        np.testing.assert_allclose(wk.compute_weights().cpu().numpy(), orc.compute_weights(0), rtol=RTOL, atol=ATOL,
                                   err_msg=f"compute weights round {t}")
        g = O.synthetic_grad(1, t, 0, n)
        wk.step(torch.from_numpy(g).cuda())
        orc.step([g])
        assert wk.round_compressed(t) == orc.compressed[t]
        assert np.array_equal(bits(wk.residual.cpu().numpy()), bits(orc.workers[0].residual)), f"residual round {t}"
    wk.flush()
    np.testing.assert_allclose(wk.weights.cpu().numpy(), orc.W, rtol=RTOL, atol=ATOL)
    for t in range(max(0, iters - 8), iters):
        assert abs(wk.grad_norm(t) - orc.grad_norms[t]) <= 1e-6 * max(1.0, orc.grad_norms[t])


@pytest.mark.parametrize("ring", [2, 4])
@pytest.mark.parametrize("sizes,k,warm", [([5000, 33], 4, 0), ([5000, 33], 3, 2), ([300_000], 2, 1)])
def test_engine_grad_norm_ring(pkg, ring, sizes, k, warm):
    # ring >= 4: the accumulating kernel zeroes the next two slots in-kernel (incl. the N=1
    # fold, which accumulates two rounds); ring < 4: a memset per round
    _, E, L, Wk = pkg
    layout = L.Layout.from_lengths(sizes)
    n = layout.total
    hp = E.HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=k, alpha=0.5, warmup_n=warm)
    w0 = O.synthetic_weights(5, n)
    wk = Wk.CDSGDWorker(layout, hp, w0, gnorm_ring=ring)
    orc = O.LockstepOracle(w0.astype(np.float64), sizes, O.OracleHP("cdsgd", 1, 0.1, 0.4, k, 0.5, warm))
    for t in range(14):
        g = O.synthetic_grad(5, t, 0, n)
        wk.step(torch.from_numpy(g).cuda())
        orc.step([g])
        if t >= 1:
            assert abs(wk.grad_norm(t - 1) - orc.grad_norms[t - 1]) <= 1e-6 * max(1.0, orc.grad_norms[t - 1]), t
    wk.flush()
    assert abs(wk.grad_norm(13) - orc.grad_norms[13]) <= 1e-6 * max(1.0, orc.grad_norms[13])


def test_engine_flush_midway_and_continue(pkg):
    _, E, L, Wk = pkg
    sizes = [2000, 17]
    layout = L.Layout.from_lengths(sizes)
    hp = E.HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=4, warmup_n=1)
    w0 = O.synthetic_weights(2, layout.total)
    wk = Wk.CDSGDWorker(layout, hp, w0)
    orc = O.LockstepOracle(w0.astype(np.float64), sizes, O.OracleHP("cdsgd", 1, 0.1, 0.4, 4, 0.5, 1))
    for t in range(12):
        g = O.synthetic_grad(2, t, 0, layout.total)
        wk.step(torch.from_numpy(g).cuda())
        orc.step([g])
        if t in (3, 7):
            wk.flush()
            np.testing.assert_allclose(wk.weights.cpu().numpy(), orc.W, rtol=RTOL, atol=ATOL)
        np.testing.assert_allclose(wk.compute_weights().cpu().numpy(), orc.compute_weights(0), rtol=RTOL, atol=ATOL)
    wk.flush()
    np.testing.assert_allclose(wk.weights.cpu().numpy(), orc.W, rtol=RTOL, atol=ATOL)


def test_engine_numeric_error_rolls_back_residual(pkg):
    from paper_2106_10796_b200.codec import CodecNumericError

    _, E, L, Wk = pkg
    sizes = [640, 100]
    layout = L.Layout.from_lengths(sizes)
    hp = E.HyperParams(algo="cdsgd", workers=1, k=4, warmup_n=0)
    wk = Wk.CDSGDWorker(layout, hp, np.zeros(layout.total, np.float32))
    for t in range(2):
        wk.step(torch.from_numpy(O.synthetic_grad(3, t, 0, layout.total)).cuda())
    wk.check()
    good = wk.residual.clone()
    g = torch.from_numpy(O.synthetic_grad(3, 2, 0, layout.total)).cuda()
    g[640 + 42] = float("nan")
    wk.step(g)  # round 2: compressed, poisoned (its apply of round 1 is valid)
    w_before, loc_before = wk.weights.clone(), wk.compute_weights().clone()
    wk.step(torch.from_numpy(O.synthetic_grad(3, 3, 0, layout.total)).cuda())  # round 3: correction
    with pytest.raises(CodecNumericError) as ei:
        wk.check()
    assert (ei.value.key, ei.value.index, ei.value.round) == (1, 42, 2)
    assert torch.equal(wk.residual, good), "residual must be the one valid before the failing round"
    # the apply of the failed round is skipped (sticky abort; small-layout kernels send those
    # stores to a sink instead of branching): W and the compute weights stay as they were
    # (bitwise: the compute weights of the poisoned round hold its NaN, loc = W - eta_l * g)
    def bits(x):
        return x.view(torch.int64 if x.dtype == torch.float64 else torch.int32)

    assert torch.equal(bits(wk.weights), bits(w_before)), "W must not move after the failing round"
    assert torch.equal(bits(wk.compute_weights()), bits(loc_before)), \
        "compute weights must not move after the failing round"
    with pytest.raises(Exception):
        wk.step(g)


# ------------------------------------------------------------------ local-sim N workers


def _abi():
    from paper_2106_10796_b200 import _lib

    return _lib.lib(), _lib


def local_sim(layout, sizes, E, name):
    lib, _lib = _abi()
    p = f"{name}_"
    nwk, k, warm, iters, seed, force, bypass = (int(x) for x in E[p + "cfg"])
    eta_g, eta_l, alpha = (float(x) for x in E[p + "hyper"])
    algo = str(E[p + "algo"])
    hp = O.OracleHP(algo, nwk, eta_g, eta_l, k, alpha, warm, bool(force), bool(bypass))
    orc = O.LockstepOracle(E[p + "w0"], sizes, hp)  # only for the schedule
    n, nw = layout.total, layout.n_words
    lay = layout.handle().ptr
    st = torch.cuda.current_stream().cuda_stream
    W = torch.from_numpy(E[p + "w0"].astype(np.float32)).cuda()
    res = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(nwk)]
    spare = torch.empty(n, dtype=torch.float64, device="cuda")
    gathered = torch.zeros(nwk * nw, dtype=torch.int32, device="cuda").view(torch.uint32)
    err = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    for t in range(iters):
        comp = orc._push_compressed(orc.workers[0])
        grads = [torch.from_numpy(E[p + "grads"][t, w]).cuda() for w in range(nwk)]
        if comp:
            for w in range(nwk):
                _lib.check(lib.cdsgd_quantize(lay, grads[w].data_ptr(), _lib.F32, res[w].data_ptr(), spare.data_ptr(),
                                              gathered.data_ptr() + 4 * w * nw, alpha, err.data_ptr(), 0, st))
                res[w], spare = spare, res[w]
            _lib.check(lib.cdsgd_apply_quant(lay, W.data_ptr(), _lib.F32, gathered.data_ptr(), nwk, nw, alpha, eta_g, None, None,
                                             eta_l, err.data_ptr(), 0, None, st))
        else:
            gsum = torch.stack(grads).sum(0)  # fp32 sum, stands in for ncclAllReduce
            _lib.check(lib.cdsgd_apply_full(W.data_ptr(), _lib.F32, gsum.data_ptr(), nwk, n, eta_g, None, None, eta_l, None, 0,
                                             None, st))
        orc.step([E[p + "grads"][t, w] for w in range(nwk)])
        np.testing.assert_allclose(W.cpu().numpy(), E[p + "weights_after"][t], rtol=RTOL, atol=ATOL,
                                   err_msg=f"{name} round {t}")
    assert [int(x) for x in err.cpu().tolist()] == [-1, -1]
    for w in range(nwk):
        assert np.array_equal(bits(res[w].cpu().numpy()), bits(E[p + "final_residual"][w])), (name, w)


@pytest.mark.parametrize("name", ["cd_n2_k4_w5", "cd_n4_k2_w1", "cd_n2_k4_w2", "cd_n8_k4_w5", "cd_n3_k4_w3",
                                  "cd_n2_force", "bit_n2", "s_n3", "cd_n2_a03"])
def test_local_sim_matches_reference_golden(pkg, engine_golden, name):
    _, _, L, _ = pkg
    sizes = [int(s) for s in engine_golden[f"{name}_sizes"]]
    local_sim(L.Layout.from_lengths(sizes), sizes, engine_golden, name)


def test_apply_quant_fused_local_update(pkg):
    """K2 with g_next: W' and loc = W' - eta_l*g_next vs fp64 oracle arithmetic."""
    lib, _lib = _abi()
    _, _, L, _ = pkg
    rng = np.random.default_rng(11)
    for nwk in (1, 2, 4, 5, 8):
        layout = L.Layout.from_lengths([5000, 33, 1024])
        n, nw = layout.total, layout.n_words
        codes = rng.integers(0, 3, size=(nwk, n)).astype(np.uint8)
        packed = np.concatenate([np.concatenate([O.pack_symbols(codes[w][layout.slice(k)]) for k in layout.keys])
                                 for w in range(nwk)])
        W = rng.standard_normal(n).astype(np.float32)
        gn = rng.standard_normal(n).astype(np.float32)
        Wd, gd = torch.from_numpy(W).cuda(), torch.from_numpy(gn).cuda()
        loc = torch.empty_like(Wd)
        gns = torch.zeros(1, dtype=torch.float64, device="cuda")
        gath = torch.from_numpy(packed.view(np.int32)).cuda().view(torch.uint32)
        err = torch.full((2,), -1, dtype=torch.int64, device="cuda")
        _lib.check(lib.cdsgd_apply_quant(layout.handle().ptr, Wd.data_ptr(), _lib.F32, gath.data_ptr(), nwk, nw, 0.5, 0.1,
                                         gd.data_ptr(), loc.data_ptr(), 0.4, err.data_ptr(), 0, gns.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream))
        deq = [O.dequantize_layout(packed[w * nw:(w + 1) * nw], 0.5, layout.lengths) for w in range(nwk)]
        mean = O.server_aggregate(deq)
        Wref = W.astype(np.float64) - 0.1 * mean
        np.testing.assert_allclose(Wd.cpu().numpy(), Wref, rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(loc.cpu().numpy(), Wref - 0.4 * gn.astype(np.float64), rtol=1e-6, atol=1e-6)
        assert abs(gns.item() - float(mean @ mean)) <= 1e-9 * max(1.0, float(mean @ mean))
        assert [int(x) for x in err.cpu().tolist()] == [-1, -1]
    # reserved symbol 11 is reported (CorruptPayloadError analogue)
    layout = L.Layout.from_lengths([600])
    words = torch.zeros(layout.n_words, dtype=torch.int32, device="cuda")
    words[3] = 3 << 10  # element 16*3 + 5
    Wd = torch.zeros(600, device="cuda")
    err = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    _lib.check(lib.cdsgd_apply_quant(layout.handle().ptr, Wd.data_ptr(), _lib.F32, words.data_ptr(), 1, layout.n_words, 0.5, 0.1,
                                     None, None, 0.4, err.data_ptr(), 0, None, torch.cuda.current_stream().cuda_stream))
    assert int(err[1].item()) == 16 * 3 + 5


def test_round_payloads_to_reference_frames(pkg):
    """The engine's codes of a round, framed for the reference PS (wire.py), carry the
    oracle's words bit for bit."""
    from paper_2106_10796_b200 import wire

    _, E, L, Wk = pkg
    sizes = [1000, 37, 16, 1]
    layout = L.Layout.from_lengths(sizes)
    hp = E.HyperParams(algo="cdsgd", workers=1, k=4, warmup_n=0)
    w0 = O.synthetic_weights(6, layout.total)
    wk = Wk.CDSGDWorker(layout, hp, w0)
    orc = O.LockstepOracle(w0.astype(np.float64), sizes, O.OracleHP("cdsgd", 1, 0.1, None, 4, 0.5, 0))
    for t in range(6):
        g = O.synthetic_grad(6, t, 0, layout.total)
        wk.step(torch.from_numpy(g).cuda())
        orc.step([g])
        if orc.compressed[t]:
            frames = wire.round_frames(0, t, payloads=wk.round_payloads(t))
            assert len(frames) == len(sizes)
            got = np.concatenate([wire.decode_frame(f).payload.words.cpu().numpy() for f in frames])
            assert np.array_equal(got, orc.words[(t, 0)]), t
        else:
            with pytest.raises(E.ConfigError):
                wk.round_payloads(t)


def test_module_integration_matches_oracle(pkg):
    """A torch MLP trained through CDSGDModule: the gradients autograd produced at the
    engine's compute weights, replayed through the lock-step oracle, give the same
    residuals (bitwise) and weights (tolerance) — the plumbing (key order, grad views,
    compute-weight reloads) is exact."""
    from paper_2106_10796_b200.model import CDSGDModule

    _, E, L, _ = pkg
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(20, 33), torch.nn.Tanh(), torch.nn.Linear(33, 3)).cuda()
    hp = E.HyperParams(algo="cdsgd", workers=1, eta_global=0.05, eta_local=0.2, k=3, alpha=0.05, warmup_n=2)
    m = CDSGDModule(net, hp)
    sizes = m.layout.lengths
    w0 = torch.cat([p.detach().reshape(-1) for p in net.parameters()]).double().cpu().numpy()
    orc = O.LockstepOracle(w0, sizes, O.OracleHP("cdsgd", 1, 0.05, 0.2, 3, 0.05, 2))
    x = torch.randn(64, 20, device="cuda")
    y = torch.randint(0, 3, (64,), device="cuda")
    for t in range(10):
        cw = torch.cat([p.detach().reshape(-1) for p in net.parameters()]).cpu().numpy()
        np.testing.assert_allclose(cw, orc.compute_weights(0), rtol=RTOL, atol=ATOL, err_msg=f"round {t}")
        torch.nn.functional.cross_entropy(net(x[t * 6:t * 6 + 6]), y[t * 6:t * 6 + 6]).backward()
        g = torch.cat([p.grad.reshape(-1) for p in net.parameters()]).cpu().numpy()
        m.step()
        orc.step([g])
        assert np.array_equal(bits(m.worker.residual.cpu().numpy()), bits(orc.workers[0].residual)), t
    m.flush()
    W = torch.cat([p.detach().reshape(-1) for p in net.parameters()]).cpu().numpy()
    np.testing.assert_allclose(W, orc.W, rtol=RTOL, atol=ATOL)


def test_engine_full_resnet50_vs_c_port(pkg):
    """The headline workload at FULL size (161 keys, 25,557,032 elements), N=1, k=4: the
    engine's residual is bitwise the reference round's (C restatement, oracle/cpu_port.py)
    after every round through two k-periods (fused, local-only, fold paths and every
    key's partial last tile), compute weights and the final W within rtol 1e-5."""
    from oracle import cpu_port

    _, E, L, Wk = pkg
    if cpu_port.load() is None:
        pytest.skip("C port not built")
    layout = L.by_name("resnet50")
    n = layout.total
    w0 = np.random.default_rng([11, 999]).standard_normal(n).astype(np.float32)
    hp = E.HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5, warmup_n=0)
    wk = Wk.CDSGDWorker(layout, hp, w0)
    port = cpu_port.CPortEngine(w0.astype(np.float64), [s.length for s in layout.spans], 1, k=4, alpha=0.5)
    for t in range(9):
        g = (0.3 * np.random.default_rng([11, t]).standard_normal(n)).astype(np.float32)
        wk.step(torch.from_numpy(g).cuda())
        port.step(g[None, :])
        assert np.array_equal(bits(wk.residual.cpu().numpy()), bits(port.res[0])), f"residual round {t}"
        np.testing.assert_allclose(wk.compute_weights().cpu().numpy(), port.loc[0], rtol=RTOL, atol=ATOL,
                                   err_msg=f"compute weights round {t}")
    wk.flush()
    np.testing.assert_allclose(wk.weights.cpu().numpy(), port.W, rtol=RTOL, atol=ATOL)
