"""Wire-format interop: frames byte-identical to the reference's
encoder (golden), and — when the reference is mounted — a worker whose pushes are
encoded by paper_2106_10796_b200.wire drives the unmodified reference ServerNode."""

import os
import sys

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O
from paper_2106_10796_b200 import codec as cx
from paper_2106_10796_b200 import wire


def test_frames_match_reference_golden(codec_golden):
    G = codec_golden
    words, _ = O.quantize(np.zeros(37), G["wire_grad"], 0.5)
    p = cx.QuantizedPayload(torch.from_numpy(words), 0.5, 37)
    vals = G["wire_vals"]
    assert wire.encode_push_quantized(3, 123456789, 7, p) == G["wire_push_quant"].tobytes()
    assert wire.encode_push_full(2, 41, 1, vals) == G["wire_push_full"].tobytes()
    assert wire.encode_push_full(2, 41, 1, torch.from_numpy(vals)) == G["wire_push_full"].tobytes()
    assert wire.encode_pull_request(5, 9) == G["wire_pull"].tobytes()
    assert wire.encode_weights(12, 3, vals) == G["wire_weights"].tobytes()
    assert wire.encode_shutdown() == G["wire_shutdown"].tobytes()
    assert wire.HEADER_BYTES == 20


def test_decode_roundtrip_and_errors(codec_golden):
    G = codec_golden
    f = wire.decode_frame(G["wire_push_quant"].tobytes(), device="cpu")
    assert (f.variant, f.worker, f.key, f.iteration) == (wire.VARIANT_PUSH_QUANTIZED, 3, 7, 123456789)
    assert f.payload.length == 37 and f.payload.threshold == 0.5
    f = wire.decode_frame(G["wire_weights"].tobytes())
    assert np.array_equal(f.payload, G["wire_vals"]) and f.key == 3 and f.iteration == 12
    assert wire.decode_frame(G["wire_shutdown"].tobytes()).variant == wire.VARIANT_SHUTDOWN
    bad = bytearray(G["wire_pull"].tobytes())
    bad[0] ^= 0xFF
    with pytest.raises(wire.ProtocolError):
        wire.decode_frame(bytes(bad))
    with pytest.raises(wire.FramingError):
        wire.decode_frame(G["wire_push_full"].tobytes()[:-1])
    with pytest.raises(wire.FramingError):
        wire.decode_frame(b"\x5d\xcd")
    with pytest.raises(wire.ProtocolError):
        wire.encode_push_full(70000, 0, 0, np.zeros(1))


def test_encoded_rounds_drive_the_reference_server():
    """Frames from wire.round_frames (codes from the oracle, i.e. what the GPU emits
    bit-for-bit) decoded by the reference protocol and folded by the reference
    ServerNode give the lock-step trajectory."""
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not mounted")
    sys.path.insert(0, src)
    sys.dont_write_bytecode = True
    try:
        import cdsgd.engine as E
        import cdsgd.protocol as P
        from cdsgd.numcore import KeyedVector, Layout as RLayout
    finally:
        sys.path.remove(src)
    from paper_2106_10796_b200.layout import Layout

    sizes, N, T = [300, 17, 64], 2, 9
    lay = Layout.from_lengths(sizes)
    rlay = RLayout([(f"k{i}", s) for i, s in enumerate(sizes)])
    w0 = O.synthetic_weights(4, lay.total).astype(np.float64)
    hp = E.HyperParams(algo="bitsgd", workers=N, eta_global=0.1, k=4, alpha=0.5, warmup_n=0, batch_size=1, iters=T)
    server = E.ServerNode(KeyedVector(w0.copy(), rlay), hp)
    orc = O.LockstepOracle(w0, sizes, O.OracleHP("bitsgd", N, 0.1, None, 4, 0.5, 0))
    res = [np.zeros(lay.total) for _ in range(N)]
    for t in range(T):
        grads = [O.synthetic_grad(4, t, w, lay.total) for w in range(N)]
        for w in range(N):
            words, res[w] = O.quantize_layout(res[w], grads[w], 0.5, sizes)
            payloads, w0i = [], 0
            for s in sizes:
                k = (s + 15) // 16
                payloads.append(cx.QuantizedPayload(torch.from_numpy(words[w0i:w0i + k].copy()), 0.5, s))
                w0i += k
            for frame in wire.round_frames(w, t, payloads=payloads):
                server.handle(P.decode_message(frame))
        orc.step(grads)
        assert np.array_equal(server.weights.values, orc.W), t
