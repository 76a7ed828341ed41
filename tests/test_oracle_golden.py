"""Pin the CPU oracle (test infrastructure) to the reference's own outputs.

The golden fixtures come from the unmodified reference (tests/golden/make_golden.py);
the SPEC known-answer tests are restated inline with their SPEC.md line numbers.
"""

import numpy as np
import pytest

from oracle import cdsgd_oracle as O


def test_spec_quantize_kats():
    # SPEC.md:122-125 (+ exact residuals from SURVEY §8c table)
    cases = [
        (0.0, 0.7, 1, 0.19999999999999996),
        (0.0, 0.0, 0, 0.0),
        (0.3, 0.1, 0, 0.4),
        (-0.2, -0.4, 2, -0.10000000000000009),
        (0.0, 0.5, 1, 0.0),    # tie emits
        (0.0, -0.5, 2, 0.0),
        (0.0, 1.7, 1, 1.2),    # one symbol even when |a| >= 2 alpha
    ]
    for r, g, sym, r_new in cases:
        w, rn = O.quantize(np.array([r]), np.array([g]), 0.5)
        assert int(w[0]) == sym
        assert rn[0] == r_new


def test_spec_pack_and_sizes():
    assert int(O.pack_symbols(np.array([1, 0, 2, 0]))[0]) == 0x21
    assert O.pack_symbols(np.zeros(0)).shape == (0,)
    assert O.payload_bytes(0) == 0 and O.payload_bytes(16) == 4 and O.payload_bytes(17) == 8
    assert O.compression_ratio(16) == 16.0 and O.compression_ratio(17) == 8.5
    assert O.compression_ratio(0) == 1.0
    # SPEC.md:497 (corrected): 16,384 elements -> 1,024 words = 4,096 B (+13)
    assert O.payload_bytes(16384) == 4096 and O.serialized_payload_bytes(16384) == 4109


def test_spec_should_compress():
    assert [O.should_compress(c, 4) for c in (1, 2, 3, 4)] == [True, True, True, False]
    assert not any(O.should_compress(c, 1) for c in range(1, 30))
    assert sum(O.should_compress(c, 5) for c in range(1, 21)) == 16


def test_oracle_quantize_matches_reference_golden(codec_golden):
    G = codec_golden
    for name in G["q_names"]:
        r, g, a = G[f"q_{name}_r"], G[f"q_{name}_g"], float(G[f"q_{name}_alpha"])
        w, rn = O.quantize(r, g, a)
        assert np.array_equal(w, G[f"q_{name}_words"]), name
        assert np.array_equal(rn.view(np.uint64), G[f"q_{name}_rnew"].view(np.uint64)), name
        deq = O.dequantize(w, a, r.shape[0])
        assert np.array_equal(deq.view(np.uint64), G[f"q_{name}_deq"].view(np.uint64)), name
        assert O.payload_to_bytes(w, a, r.shape[0]) == G[f"q_{name}_bytes"].tobytes(), name
        w2, a2, n2 = O.payload_from_bytes(G[f"q_{name}_bytes"].tobytes())
        assert np.array_equal(w2, w) and a2 == a and n2 == r.shape[0]


def test_oracle_stream_matches_reference(codec_golden):
    G = codec_golden
    r = np.zeros(G["stream_g"].shape[1])
    for t in range(G["stream_g"].shape[0]):
        w, r = O.quantize(r, G["stream_g"][t], 0.5)
        assert np.array_equal(w, G["stream_words"][t])
        assert np.array_equal(r.view(np.uint64), G["stream_r"][t].view(np.uint64))


def test_oracle_errors_match_reference(codec_golden):
    G = codec_golden
    for name in G["e_names"]:
        with pytest.raises(O.OracleNumericError) as ei:
            O.quantize(G[f"e_{name}_r"], G[f"e_{name}_g"], 0.5)
        assert ei.value.index == int(G[f"e_{name}_index"])
    with pytest.raises(O.OracleCorruptPayload) as ei:
        O.dequantize(G["corrupt_words"], 0.5, int(G["corrupt_length"]))
    assert str(ei.value) == str(G["corrupt_msg"])
    assert np.array_equal(O.dequantize(np.array([0xC0000000], np.uint32), 0.5, 15), G["padbits_deq"])


def test_oracle_pack_matches_reference(codec_golden):
    G = codec_golden
    assert np.array_equal(O.pack_symbols(np.array([1, 0, 2, 0])), G["pack_kat"])
    assert np.array_equal(O.pack_symbols(G["pack_syms"]), G["pack_words"])
    assert np.array_equal(O.unpack_symbols(G["pack_words"], 1001), G["pack_syms"])


def _engine_case(E, name):
    p = f"{name}_"
    n_workers, k, warmup, iters, seed, force, bypass = (int(x) for x in E[p + "cfg"])
    eta_g, eta_l, alpha = (float(x) for x in E[p + "hyper"])
    hp = O.OracleHP(algo=str(E[p + "algo"]), workers=n_workers, eta_global=eta_g, eta_local=eta_l,
                    k=k, alpha=alpha, warmup_n=warmup, force_compress=bool(force),
                    bypass_local=bool(bypass))
    return hp, [int(s) for s in E[p + "sizes"]], iters


def test_oracle_engine_matches_reference_bitwise(engine_golden):
    E = engine_golden
    for name in E["names"]:
        p = f"{name}_"
        hp, sizes, iters = _engine_case(E, name)
        orc = O.LockstepOracle(E[p + "w0"], sizes, hp)
        for t in range(iters):
            for w in range(hp.workers):
                cw = orc.compute_weights(w)
                assert np.array_equal(cw, E[p + "compute"][t, w]), (name, t, w)
            orc.step(list(E[p + "grads"][t]))
            assert np.array_equal(orc.W, E[p + "weights_after"][t]), (name, t)
        assert orc.compressed == [bool(x) for x in E[p + "compressed"]], name
        for w in range(hp.workers):
            assert np.array_equal(orc.workers[w].residual, E[p + "final_residual"][w]), name
        np.testing.assert_allclose(orc.grad_norms, E[p + "grad_norm"], rtol=1e-12)


def test_compressed_flag_pattern(engine_golden):
    # warm-up 5, k=4 -> 00000 1110 1110 ...
    pat = "".join("1" if c else "0" for c in engine_golden["cd_n2_k4_w5_compressed"])
    assert pat == "0000011101110111"


def test_oracle_matches_live_reference_if_present():
    """Optional: re-check against the live reference when it is mounted (build container)."""
    import os
    import sys

    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not mounted")
    sys.path.insert(0, src)
    sys.dont_write_bytecode = True
    try:
        import cdsgd.codec as codec
    finally:
        sys.path.remove(src)
    rng = np.random.default_rng(99)
    for n in (1, 16, 17, 2049):
        r = rng.standard_normal(n) * 0.4
        g = (rng.standard_normal(n) * 0.6).astype(np.float32)
        st = codec.ResidualState(r.copy())
        p, st = codec.quantize(st, g, 0.5)
        w, rn = O.quantize(r, g, 0.5)
        assert np.array_equal(w, p.words) and np.array_equal(rn, st.residual)
