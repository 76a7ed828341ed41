"""Generate golden vectors from the UNMODIFIED reference (cdsgd 0.1.0).

Run in the build container only (the reference does not travel to the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``cdsgd`` from ``/root/reference/pkg/src`` and writes

* ``codec_golden.npz``  — ``codec.quantize`` / ``dequantize`` / ``pack_symbols`` cases
  (codec.py:140-206), including ties, signed zeros, |a| >= 2*alpha, subnormals,
  non-finite error indices and reserved-symbol error indices;
* ``costmodel_golden.npz`` — the time model (costmodel.py:51-152) over a grid of
  timing constants (``--only-costmodel`` regenerates just this file);
* ``engine_golden.npz`` — lock-step engine traces (engine.py:614-663) on synthetic
  gradients: ``loss_and_grad`` (engine.py:363) is the ONLY thing replaced, by a
  function that returns the pre-drawn gradient for call (t, w); Worker,
  ServerNode and _run_lockstep run unmodified (SURVEY §8c recipe).

The fixtures are small (< 1 MB) and committed; tests never need the reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import cdsgd.codec as codec  # noqa: E402
import cdsgd.engine as engine  # noqa: E402
from cdsgd.numcore import Dataset, KeyedVector, Layout, ModelSpec  # noqa: E402


def synthetic_grad(seed, t, w, n, scale=0.3):
    rng = np.random.default_rng([seed, t, w])
    return (scale * rng.standard_normal(n)).astype(np.float32)


def synthetic_weights(seed, n):
    return np.random.default_rng([seed, 999]).standard_normal(n).astype(np.float32)


def codec_cases():
    out = {}
    cases = []
    rng = np.random.default_rng(1234)
    # (name, residual f64, grad (f32 or f64), alpha)
    for n in (0, 1, 15, 16, 17, 31, 33, 100, 1000, 4099):
        r = (0.4 * rng.standard_normal(n)).astype(np.float64)
        g = (0.5 * rng.standard_normal(n)).astype(np.float32)
        cases.append((f"rand{n}", r, g, 0.5))
    n = 777
    cases.append(("alpha0.3", 0.2 * rng.standard_normal(n), (0.3 * rng.standard_normal(n)).astype(np.float32), 0.3))
    cases.append(("alpha1e-3", 1e-3 * rng.standard_normal(n), (1e-3 * rng.standard_normal(n)).astype(np.float32), 1e-3))
    cases.append(("g64", 0.3 * rng.standard_normal(n), 0.7 * rng.standard_normal(n), 0.5))
    special_r = np.array([0.0, 0.0, 0.3, -0.2, 0.0, 0.0, -0.0, 0.0, 0.25, -0.25, 1e-310, -1e-310, 0.0, 0.0, 0.5, -0.5, 0.0], dtype=np.float64)
    special_g = np.array([0.7, 0.0, 0.1, -0.4, 0.5, -0.5, -0.0, 1.7, 0.25, -0.25, 0.0, 0.0, -1.7, 3.0, 0.0, 0.0, 1e-45], dtype=np.float32)
    cases.append(("special", special_r, special_g, 0.5))
    # A multi-step stream: the residual carried across 60 steps on one key.
    rs = np.zeros(300)
    stream_g = []
    stream_w = []
    stream_r = []
    for t in range(60):
        g = synthetic_grad(7, t, 0, 300)
        st = codec.ResidualState(rs.copy())
        p, st = codec.quantize(st, g, 0.5)
        rs = st.residual.copy()
        stream_g.append(g)
        stream_w.append(p.words.copy())
        stream_r.append(rs.copy())
    out["stream_g"] = np.stack(stream_g)
    out["stream_words"] = np.stack(stream_w)
    out["stream_r"] = np.stack(stream_r)

    names = []
    for name, r, g, alpha in cases:
        st = codec.ResidualState(np.array(r, dtype=np.float64, copy=True))
        p, st2 = codec.quantize(st, g, alpha)
        out[f"q_{name}_r"] = np.asarray(r, dtype=np.float64)
        out[f"q_{name}_g"] = g
        out[f"q_{name}_alpha"] = np.float64(alpha)
        out[f"q_{name}_words"] = p.words
        out[f"q_{name}_rnew"] = st2.residual
        out[f"q_{name}_deq"] = codec.dequantize(p)
        out[f"q_{name}_bytes"] = np.frombuffer(p.to_bytes(), dtype=np.uint8)
        names.append(name)
    out["q_names"] = np.array(names)

    # Non-finite error index (codec.py:181-185): residual must stay untouched.
    errs = []
    for name, g in [
        ("inf1", np.array([0.0, np.inf, np.nan], dtype=np.float32)),
        ("nan_late", np.concatenate([np.zeros(40, np.float32), [np.nan], np.zeros(5, np.float32)])),
        ("ninf0", np.array([-np.inf] + [0.1] * 20, dtype=np.float32)),
    ]:
        r0 = np.linspace(-0.4, 0.4, g.shape[0])
        st = codec.ResidualState(r0.copy())
        try:
            codec.quantize(st, g, 0.5)
            raise AssertionError("expected CodecNumericError")
        except codec.CodecNumericError as exc:
            assert np.array_equal(st.residual, r0)
            out[f"e_{name}_g"] = g
            out[f"e_{name}_r"] = r0
            out[f"e_{name}_index"] = np.int64(exc.index)
            errs.append(name)
    out["e_names"] = np.array(errs)

    # Reserved symbol 11 (codec.py:200-202): first offending element index.
    bad_words = np.array([0x00000021, 0x0000C000, 0xFFFFFFFF], dtype=np.uint32)
    try:
        codec.dequantize(codec.QuantizedPayload(bad_words, 0.5, 40))
        raise AssertionError("expected CorruptPayloadError")
    except codec.CorruptPayloadError as exc:
        out["corrupt_words"] = bad_words
        out["corrupt_length"] = np.int64(40)
        out["corrupt_msg"] = np.array(str(exc))
    # Pad bits beyond `length` are NOT validated (probe in SURVEY §8a row a3).
    pad_words = np.array([0xC0000000], dtype=np.uint32)
    out["padbits_deq"] = codec.dequantize(codec.QuantizedPayload(pad_words, 0.5, 15))

    # pack/unpack: SPEC.md:141 and random round trip.
    out["pack_kat"] = codec.pack_symbols(np.array([1, 0, 2, 0], dtype=np.uint8))
    syms = rng.integers(0, 3, size=1001).astype(np.uint8)
    out["pack_syms"] = syms
    out["pack_words"] = codec.pack_symbols(syms)
    return out


def engine_trace(name, sizes, n_workers, algo, k, warmup, iters, seed=0, eta_g=0.1, eta_l=0.4,
                 alpha=0.5, force_compress=False, bypass_local=False):
    layout = Layout([(f"k{i}", s) for i, s in enumerate(sizes)])
    n = layout.total
    w0 = synthetic_weights(seed, n).astype(np.float64)
    grads = np.stack([
        np.stack([synthetic_grad(seed, t, w, n) for w in range(n_workers)]) for t in range(iters)
    ])  # [T, N, n] float32
    calls = {"c": 0}

    def fake_loss_and_grad(model, weights, X, y):
        t, w = divmod(calls["c"], n_workers)
        calls["c"] += 1
        return 0.0, KeyedVector(grads[t, w].astype(np.float64), layout)

    saved = engine.loss_and_grad
    engine.loss_and_grad = fake_loss_and_grad
    try:
        hp = engine.HyperParams(algo=algo, workers=n_workers, eta_global=eta_g, eta_local=eta_l,
                                k=k, alpha=alpha, warmup_n=warmup, batch_size=1, iters=iters,
                                seed=seed).validate()
        trace = engine.RunTrace(weights=True, grads=True, compute=True, emissions=True, means=True)
        init = KeyedVector(w0.copy(), layout)
        server = engine.ServerNode(init, hp, trace=trace)
        ds = Dataset(np.zeros((n_workers, 1)), np.zeros(n_workers)).with_shards(n_workers)
        rngs = [np.random.default_rng(i) for i in range(n_workers)]
        workers = [
            engine.Worker(w, ModelSpec("linear-regression", 1, 1), ds, hp, init, rngs[w], trace=trace,
                          force_compress=force_compress, bypass_local=bypass_local)
            for w in range(n_workers)
        ]
        rounds = engine._run_lockstep(server, workers, iters, layout)
        for w in workers:
            w.snapshot_residuals(trace)
    finally:
        engine.loss_and_grad = saved
    p = f"{name}_"
    out = {
        p + "sizes": np.array(sizes, dtype=np.int64),
        p + "cfg": np.array([n_workers, k, warmup, iters, seed, int(force_compress), int(bypass_local)], dtype=np.int64),
        p + "algo": np.array(algo),
        p + "hyper": np.array([eta_g, eta_l, alpha]),
        p + "w0": w0,
        p + "grads": grads,
        p + "weights_after": np.stack([trace.weights_after[t] for t in range(iters)]),
        p + "compute": np.stack([np.stack([trace.compute_weights[(t, w)] for w in range(n_workers)])
                                  for t in range(iters)]),
        p + "compressed": np.array([trace.compressed_rounds[t] for t in range(iters)]),
        p + "grad_norm": np.array(server.grad_norms),
        p + "bytes": np.array([sum(r.bytes_pushed for r in rnd) for rnd in rounds], dtype=np.int64),
        p + "final_residual": np.stack([
            np.concatenate([trace.final_residuals[(w, key)] for key in range(len(sizes))])
            for w in range(n_workers)
        ]),
    }
    return out


ENGINE_CASES = [
    # name, sizes, N, algo, k, warmup, iters, extra
    ("cd_n2_k4_w5", [1000, 37, 16, 1], 2, "cdsgd", 4, 5, 16, {}),
    ("cd_n1_k3_w0", [300], 1, "cdsgd", 3, 0, 10, {}),
    ("cd_n4_k2_w1", [64, 17], 4, "cdsgd", 2, 1, 9, {}),
    ("cd_n2_k4_w2", [513], 2, "cdsgd", 4, 2, 12, {}),
    ("cd_n8_k4_w5", [200, 56], 8, "cdsgd", 4, 5, 12, {}),
    ("cd_n3_k4_w3", [129, 3, 64], 3, "cdsgd", 4, 3, 10, {}),
    ("cd_n2_k1_w2", [90], 2, "cdsgd", 1, 2, 6, {}),
    ("cd_n2_force", [150], 2, "cdsgd", 4, 2, 8, {"force_compress": True}),
    ("cd_n2_bypass", [150], 2, "cdsgd", 4, 0, 8, {"bypass_local": True}),
    ("bit_n2", [100, 28], 2, "bitsgd", 5, 5, 6, {}),
    ("lu_n2_w2", [100, 28], 2, "lusgd", 5, 2, 6, {}),
    ("s_n3", [77], 3, "ssgd", 5, 5, 5, {}),
    ("cd_n2_a03", [400], 2, "cdsgd", 4, 1, 10, {"alpha": 0.3, "eta_g": 0.05, "eta_l": 0.2}),
]


def wire_cases():
    """Frames of every variant from the reference encoder (protocol.py:116-140)."""
    import cdsgd.protocol as protocol

    rng = np.random.default_rng(77)
    g = (0.6 * rng.standard_normal(37)).astype(np.float32)
    payload, _ = codec.quantize(codec.ResidualState.zeros(37), g, 0.5)
    vals = rng.standard_normal(5)
    msgs = {
        "push_quant": protocol.PushQuantized(3, 123456789, 7, payload),
        "push_full": protocol.PushFull(2, 41, 1, vals),
        "pull": protocol.PullRequest(5, 9),
        "weights": protocol.Weights(12, 3, vals),
        "shutdown": protocol.Shutdown(),
    }
    out = {"wire_grad": g, "wire_vals": vals}
    for name, m in msgs.items():
        out[f"wire_{name}"] = np.frombuffer(protocol.encode_message(m), dtype=np.uint8)
    return out


def costmodel_cases():
    """Eq. 6-9 over a grid of timing constants that hits every case and the ties
    (costmodel.py:51-152): averages, per-iteration comm / time / savings, regime, and
    the cumulative timeline."""
    import itertools
    import warnings

    import cdsgd.costmodel as cm

    vals = (0.0, 0.5, 1.0, 1.5, 3.0)
    params, avg, per_i, regime, cum = [], [], [], [], []
    for tau, phi, psi, delta in itertools.product(vals, vals, vals, (0.0, 0.25, 1.0)):
        for k in (1, 2, 4, 5):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                p = cm.CostParams(tau=tau, phi=phi, psi=psi, delta=delta, k=k)
            params.append((tau, phi, psi, delta, k))
            avg.append((cm.t_ssgd(p), cm.t_loc(p), cm.t_bit(p), cm.avg_cd(p)))
            rows = []
            for i in range(1, 11):
                rows.append((cm.comm_cd(i, p), cm.t_cd(i, p), cm.saving_vs_loc(i, p), cm.saving_vs_bit(i, p)))
            per_i.append(rows)
            regime.append(cm.classify_regime(p))
            tl = cm.timeline(p, 10)
            cum.append([r[3] for r in tl])
    return {"cm_params": np.array(params, dtype=np.float64), "cm_avg": np.array(avg),
            "cm_per_i": np.array(per_i), "cm_regime": np.array(regime), "cm_timeline_cum": np.array(cum)}


def main():
    if "--only-costmodel" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "costmodel_golden.npz"), **costmodel_cases())
        print("wrote costmodel_golden.npz")
        return
    np.savez_compressed(os.path.join(HERE, "costmodel_golden.npz"), **costmodel_cases())
    codec_out = codec_cases()
    codec_out.update(wire_cases())
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), **codec_out)
    eng = {}
    names = []
    for name, sizes, n, algo, k, w, it, extra in ENGINE_CASES:
        eng.update(engine_trace(name, sizes, n, algo, k, w, it, **extra))
        names.append(name)
    eng["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "engine_golden.npz"), **eng)
    print("wrote", len(codec_out), "codec arrays and", len(names), "engine traces")


if __name__ == "__main__":
    main()
