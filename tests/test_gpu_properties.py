"""SPEC properties of the codec and the engine, checked on the GPU path at the sizes the
reference's acceptance criteria name.

* Acceptance 1: codec conservation — 1,000 gradient streams of length 256
  (one key each: the GPU quantizes them as ONE 1,000-key layout), T = 200 steps, α = 0.5:
  Σ_t dequantize(q_t) + r_T = Σ_t g_t per coordinate, relative error < 1e-10.
* Sign consistency and dead zone on every element of every step.
* Packing bijection on well-formed symbols.
* Acceptance 4(a): cdsgd with k = 1 and η_l = η_g is lusgd — bitwise, on the
  engine (N = 1), every round.
"""

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2106_10796_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)
    return _lib


def test_conservation_1000_streams_200_steps(L):
    from paper_2106_10796_b200.layout import Layout

    K, n_k, T, alpha = 1000, 256, 200, 0.5
    lay = Layout.from_lengths([n_k] * K)
    n, nw = lay.total, lay.n_words
    st = torch.cuda.current_stream().cuda_stream
    gen = torch.Generator(device="cuda").manual_seed(496)
    r = [torch.zeros(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")]
    words = torch.zeros(nw, dtype=torch.int32, device="cuda")
    deq = torch.empty(n, dtype=torch.float64, device="cuda")
    sum_g = torch.zeros(n, dtype=torch.float64, device="cuda")
    sum_e = torch.zeros(n, dtype=torch.float64, device="cuda")
    err = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    cur = 0
    for t in range(T):
        g = torch.randn(n, device="cuda", generator=gen) * 0.4
        acc = r[cur] + g.double()
        L.check(L.lib().cdsgd_quantize(lay.handle().ptr, g.data_ptr(), L.F32, r[cur].data_ptr(), r[cur ^ 1].data_ptr(),
                                       words.data_ptr(), alpha, err.data_ptr(), 0, st))
        L.check(L.lib().cdsgd_dequantize_sum(lay.handle().ptr, words.data_ptr(), 1, nw, alpha, deq.data_ptr(),
                                             err.data_ptr(), st))
        cur ^= 1
        # sign consistency + dead zone
        nz = deq != 0
        assert bool(torch.all(torch.sign(deq[nz]) == torch.sign(acc[nz])))
        assert bool(torch.all(acc[nz].abs() >= alpha))
        assert bool(torch.all(r[cur][~nz].abs() < alpha)) and bool(torch.equal(r[cur][~nz], acc[~nz]))
        sum_g += g.double()
        sum_e += deq
    assert [int(x) for x in err.cpu().tolist()] == [-1, -1]
    lhs, rhs = sum_e + r[cur], sum_g
    rel = ((lhs - rhs).abs() / rhs.abs().clamp_min(1e-300)).max().item()
    absd = (lhs - rhs).abs().max().item()
    assert rel < 1e-10 or absd < 1e-12, (rel, absd)


def test_pack_roundtrip_bijection(L):
    from paper_2106_10796_b200 import codec

    rng = np.random.default_rng(158)
    for n in (1, 15, 16, 17, 1000, 65537):
        sym = rng.integers(0, 3, n).astype(np.uint8)
        words = codec.pack_symbols(torch.from_numpy(sym).cuda())
        back = codec.unpack_symbols(words, n)
        assert np.array_equal(np.asarray(back.cpu()), sym)
        assert np.array_equal(words.view(torch.int32).cpu().numpy().view(np.uint32), O.pack_symbols(sym))


@pytest.mark.parametrize("weights", ["f64", "f32"])
def test_cdsgd_k1_is_lusgd_bitwise(L, weights):
    """SPEC acceptance 4(a): cdsgd with k=1 (every round a correction) and eta_l = eta_g is
    lusgd, bit for bit, through the engine."""
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import Layout
    from paper_2106_10796_b200.worker import CDSGDWorker

    sizes = [4099, 512, 3]
    lay = Layout.from_lengths(sizes)
    n = lay.total
    w0 = O.synthetic_weights(9, n)
    a = CDSGDWorker(lay, HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.1, k=1, warmup_n=2), w0,
                    weights=weights)
    b = CDSGDWorker(lay, HyperParams(algo="lusgd", workers=1, eta_global=0.1, eta_local=0.1, k=1, warmup_n=2), w0,
                    weights=weights)
    for t in range(40):
        g = torch.from_numpy(O.synthetic_grad(9, t, 0, n)).cuda()
        a.step(g)
        b.step(g)
        assert torch.equal(a.compute_weights(), b.compute_weights()), t
    a.flush()
    b.flush()
    assert torch.equal(a.weights, b.weights)
