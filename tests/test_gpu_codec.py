"""GPU parity of the codec kernels (K1 quantize, dequantize, pack/unpack, aggregate,
updates) against the reference golden vectors and the CPU oracle — bit-exact for
codes and fp64 residuals. All calls go through the C ABI (libcdsgd_b200.so)."""

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cx():
    from paper_2106_10796_b200 import _lib, codec

    _lib.load()
    torch.cuda.set_device(0)
    return codec


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a.view(np.uint32)


def run_q(cx, r, g, alpha):
    st = cx.ResidualState(torch.from_numpy(np.asarray(r, np.float64)).cuda())
    p, st = cx.quantize(st, torch.from_numpy(np.asarray(g)).cuda(), alpha)
    return p.words.cpu().numpy(), st.residual.cpu().numpy(), p


def test_quantize_golden(cx, codec_golden):
    G = codec_golden
    for name in G["q_names"]:
        r, g, a = G[f"q_{name}_r"], G[f"q_{name}_g"], float(G[f"q_{name}_alpha"])
        w, rn, p = run_q(cx, r, g, a)
        assert np.array_equal(w, G[f"q_{name}_words"]), name
        assert np.array_equal(bits(rn), bits(G[f"q_{name}_rnew"])), name
        assert p.to_bytes() == G[f"q_{name}_bytes"].tobytes(), name
        deq = cx.dequantize(p).cpu().numpy()
        assert np.array_equal(bits(deq), bits(G[f"q_{name}_deq"])), name


def test_quantize_stream_golden(cx, codec_golden):
    G = codec_golden
    st = cx.ResidualState.zeros(G["stream_g"].shape[1])
    for t in range(G["stream_g"].shape[0]):
        p, st = cx.quantize(st, torch.from_numpy(G["stream_g"][t]).cuda(), 0.5)
        assert np.array_equal(p.words.cpu().numpy(), G["stream_words"][t]), t
        assert np.array_equal(bits(st.residual.cpu().numpy()), bits(G["stream_r"][t])), t


def test_quantize_errors_golden(cx, codec_golden):
    G = codec_golden
    for name in G["e_names"]:
        r0 = G[f"e_{name}_r"]
        st = cx.ResidualState(torch.from_numpy(r0).cuda())
        with pytest.raises(cx.CodecNumericError) as ei:
            cx.quantize(st, torch.from_numpy(G[f"e_{name}_g"]).cuda(), 0.5)
        assert ei.value.index == int(G[f"e_{name}_index"])
        assert np.array_equal(bits(st.residual.cpu().numpy()), bits(r0)), "residual must be untouched"
    with pytest.raises(cx.CorruptPayloadError):
        cx.dequantize(cx.QuantizedPayload(torch.from_numpy(G["corrupt_words"]).cuda(), 0.5, int(G["corrupt_length"])))
    try:
        cx.dequantize(cx.QuantizedPayload(torch.from_numpy(G["corrupt_words"]).cuda(), 0.5, int(G["corrupt_length"])))
    except cx.CorruptPayloadError as exc:
        assert str(exc) == str(G["corrupt_msg"])
    pad = cx.dequantize(cx.QuantizedPayload(torch.tensor([0xC0000000], dtype=torch.uint32).cuda(), 0.5, 15))
    assert np.array_equal(pad.cpu().numpy(), G["padbits_deq"])
    with pytest.raises(cx.CodecError):
        cx.quantize(cx.ResidualState.zeros(4), torch.zeros(4).cuda(), 0.0)
    with pytest.raises(cx.CodecError):
        cx.quantize(cx.ResidualState.zeros(4), torch.zeros(5).cuda(), 0.5)


def test_pack_unpack_golden(cx, codec_golden):
    G = codec_golden
    assert np.array_equal(cx.pack_symbols(np.array([1, 0, 2, 0], np.uint8)).cpu().numpy(), G["pack_kat"])
    w = cx.pack_symbols(torch.from_numpy(G["pack_syms"]).cuda())
    assert np.array_equal(w.cpu().numpy(), G["pack_words"])
    assert np.array_equal(cx.unpack_symbols(w, 1001).cpu().numpy(), G["pack_syms"])
    assert cx.pack_symbols(np.zeros(0, np.uint8)).numel() == 0
    with pytest.raises(cx.CorruptPayloadError):
        cx.pack_symbols(np.array([0, 1, 3], np.uint8))
    with pytest.raises(cx.CodecError):
        cx.unpack_symbols(w, 16 * w.numel() + 1)


@pytest.mark.parametrize("n", [1, 15, 16, 17, 127, 128, 511, 512, 513, 4096 + 5, 1 << 20, (1 << 20) + 3])
def test_quantize_random_vs_oracle(cx, n):
    rng = np.random.default_rng(n)
    r = rng.standard_normal(n) * 0.4
    g = (rng.standard_normal(n) * 0.6).astype(np.float32)
    w, rn, _ = run_q(cx, r, g, 0.5)
    ow, orn = O.quantize(r, g, 0.5)
    assert np.array_equal(w, ow)
    assert np.array_equal(bits(rn), bits(orn))


def test_quantize_misaligned_views(cx):
    """Views starting off a 32-byte boundary take the coalesced ballot path."""
    n = 5000
    rng = np.random.default_rng(5)
    base_g = torch.from_numpy((rng.standard_normal(n + 3) * 0.6).astype(np.float32)).cuda()
    base_r = torch.from_numpy(rng.standard_normal(n + 3) * 0.4).cuda()
    for off in (1, 2, 3):
        g = base_g[off:off + n]
        st = cx.ResidualState(base_r[off:off + n])
        p, st = cx.quantize(st, g, 0.5)
        ow, orn = O.quantize(base_r[off:off + n].cpu().numpy(), g.cpu().numpy(), 0.5)
        assert np.array_equal(p.words.cpu().numpy(), ow)
        assert np.array_equal(bits(st.residual.cpu().numpy()), bits(orn))


LAYOUTS = {
    "two_key_unaligned": [1048575, 1],
    "odd": [3, 1000, 5, 16, 17, 1, 513, 2048, 31],
    "tiny": [1, 1, 1, 2],
}


@pytest.mark.parametrize("name", list(LAYOUTS) + ["resnet20", "resnet50"])
def test_quantize_keys_vs_oracle(cx, name):
    from paper_2106_10796_b200.layout import Layout, by_name

    layout = by_name(name) if name in ("resnet20", "resnet50") else Layout.from_lengths(LAYOUTS[name])
    n = layout.total
    rng = np.random.default_rng(17)
    r = rng.standard_normal(n) * 0.3
    g = (rng.standard_normal(n) * 0.5).astype(np.float32)
    st = cx.ResidualState(torch.from_numpy(r).cuda())
    payloads, words, st = cx.quantize_keys(st, torch.from_numpy(g).cuda(), 0.5, layout)
    ow, orn = O.quantize_layout(r, g, 0.5, layout.lengths)
    assert np.array_equal(words.cpu().numpy(), ow)
    assert np.array_equal(bits(st.residual.cpu().numpy()), bits(orn))
    assert len(payloads) == len(layout)
    assert sum(p.nbytes for p in payloads) == sum(13 + 4 * ((s + 15) // 16) for s in layout.lengths)


def test_quantize_keys_error_reports_key_local_index(cx):
    from paper_2106_10796_b200.layout import Layout

    layout = Layout.from_lengths([100, 50, 600])
    g = torch.zeros(750, dtype=torch.float32)
    g[100 + 37] = float("nan")
    g[100 + 600 - 1 + 50] = float("inf")
    st = cx.ResidualState.zeros(750)
    with pytest.raises(cx.CodecNumericError) as ei:
        cx.quantize_keys(st, g.cuda(), 0.5, layout)
    assert ei.value.key == 1 and ei.value.index == 37


def test_residual_carried_100_steps_1m(cx):
    """SURVEY §7 minimum slice: 1M elements, 100 successive steps, bitwise."""
    n = 1 << 20
    st = cx.ResidualState.zeros(n)
    r = np.zeros(n)
    for t in range(100):
        g = O.synthetic_grad(0, t, 0, n)
        p, st = cx.quantize(st, torch.from_numpy(g).cuda(), 0.5)
        w, r = O.quantize(r, g, 0.5)
        if t % 9 == 0 or t == 99:
            assert np.array_equal(p.words.cpu().numpy(), w), t
            assert np.array_equal(bits(st.residual.cpu().numpy()), bits(r)), t
    assert np.array_equal(bits(st.residual.cpu().numpy()), bits(r))


def test_server_aggregate_and_updates(cx):
    from paper_2106_10796_b200 import engine as E
    from paper_2106_10796_b200.layout import Layout

    n = 3001
    rng = np.random.default_rng(3)
    for nw in (1, 2, 3, 4, 7, 8):
        payloads, ref = {}, []
        for w in range(nw):
            r = rng.standard_normal(n) * 0.3
            g = (rng.standard_normal(n) * 0.5).astype(np.float32)
            p, _ = cx.quantize(cx.ResidualState(torch.from_numpy(r).cuda()), torch.from_numpy(g).cuda(), 0.3)
            payloads[w] = ("quant", p)
            ow, _ = O.quantize(r, g, 0.3)
            ref.append(O.dequantize(ow, 0.3, n))
        got = E.server_aggregate(dict(reversed(list(payloads.items()))), nw).cpu().numpy()
        assert np.array_equal(bits(got), bits(O.server_aggregate(ref))), nw
        fulls = [rng.standard_normal(n).astype(np.float32) for _ in range(nw)]
        got = E.server_aggregate({w: ("full", torch.from_numpy(f).cuda()) for w, f in enumerate(fulls)}, nw)
        assert np.array_equal(bits(got.cpu().numpy()), bits(O.server_aggregate(fulls))), nw
    with pytest.raises(E.ProtocolViolation):
        E.server_aggregate({0: ("full", torch.zeros(3).cuda())}, 2)
    with pytest.raises(E.ProtocolViolation):
        E.server_aggregate({0: ("full", torch.zeros(3).cuda()), 1: ("quant", None)}, 2)
    lay = Layout.from_lengths([1000, 2001])
    W = rng.standard_normal(n)
    M = rng.standard_normal(n)
    kv = E.KeyedVector(W.copy(), lay)
    E.global_update(kv, E.KeyedVector(M, lay), 0.1)
    assert np.array_equal(bits(kv.values.cpu().numpy()), bits(O.global_update(W.copy(), M, 0.1)))
    G = rng.standard_normal(n).astype(np.float32)
    loc = E.local_update(E.KeyedVector(W, lay), E.KeyedVector(torch.from_numpy(G).cuda(), lay), 0.4)
    assert np.array_equal(bits(loc.values.cpu().numpy()), bits(O.local_update(W, G, 0.4)))
