"""CPU oracle for the CD-SGD hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it. The product path
(``paper_2106_10796_b200``) never imports anything under ``oracle/`` and fails
loudly when its CUDA extension is missing.

It is a NumPy restatement of the reference algorithm (reference package
``cdsgd`` 0.1.0, ``/root/reference/pkg/src/cdsgd``), written from its behaviour,
every function citing the reference file:line it follows. Arithmetic is fp64
exactly as in the reference (``codec.py:176`` casts the gradient to float64,
``numcore.py:95`` keeps every KeyedVector in float64), so codes and residuals
from this oracle are bitwise the reference's.

Parity pin: ``tests/golden/*.npz`` were produced by the *unmodified* reference
(``tests/golden/make_golden.py`` imports it from ``/root/reference``), and
``tests/test_oracle_golden.py`` checks this oracle against every one of them
plus the SPEC known-answer tests (SPEC.md:122-125,141-143,150-152,163-164,
265-267).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

SYM_ZERO, SYM_PLUS, SYM_MINUS = 0, 1, 2          # codec.py:22-24
SYMBOLS_PER_WORD = 16                             # codec.py:25
CODEC_TAG = 0x02                                  # codec.py:28
_HEADER = struct.Struct("<BdI")                   # codec.py:29
PAYLOAD_HEADER_BYTES = _HEADER.size               # 13, codec.py:30


class OracleNumericError(ArithmeticError):
    """Mirror of codec.CodecNumericError (codec.py:41-46)."""

    def __init__(self, message: str, index: int):
        super().__init__(message)
        self.index = index


class OracleCorruptPayload(ValueError):
    """Mirror of codec.CorruptPayloadError (codec.py:33-34)."""


# ----------------------------------------------------------------------------- codec


def words_needed(n: int) -> int:
    """ceil(n/16) — codec.py:49-50."""
    return (n + SYMBOLS_PER_WORD - 1) // SYMBOLS_PER_WORD


def payload_bytes(n: int) -> int:
    """4*ceil(n/16) — codec.py:53-57."""
    if n < 0:
        raise ValueError("element count must be >= 0")
    return 4 * words_needed(n)


def compression_ratio(n: int) -> float:
    """codec.py:60-64."""
    return 1.0 if n == 0 else (4.0 * n) / payload_bytes(n)


def serialized_payload_bytes(n: int) -> int:
    """codec.py:67-69."""
    return PAYLOAD_HEADER_BYTES + payload_bytes(n)


def pack_symbols(symbols: np.ndarray) -> np.ndarray:
    """Symbol j -> bits 2(j%16)..+1 of word j//16, zero pad — codec.py:140-151."""
    s = np.asarray(symbols, dtype=np.uint32)
    if s.size and s.max() > SYM_MINUS:
        raise OracleCorruptPayload("symbols must be in {0, 1, 2}")
    nw = words_needed(s.shape[0])
    padded = np.zeros(nw * SYMBOLS_PER_WORD, dtype=np.uint32)
    padded[: s.shape[0]] = s
    shifts = (2 * np.arange(SYMBOLS_PER_WORD, dtype=np.uint32))[None, :]
    return np.bitwise_or.reduce(padded.reshape(nw, SYMBOLS_PER_WORD) << shifts, axis=1).astype(
        np.uint32
    )


def unpack_symbols(words: np.ndarray, length: int) -> np.ndarray:
    """Inverse of pack_symbols for the first `length` symbols — codec.py:154-161."""
    w = np.asarray(words, dtype=np.uint32)
    if length < 0 or length > w.shape[0] * SYMBOLS_PER_WORD:
        raise ValueError(f"{length} symbols do not fit in {w.shape[0]} words")
    shifts = (2 * np.arange(SYMBOLS_PER_WORD, dtype=np.uint32))[None, :]
    return ((w[:, None] >> shifts) & np.uint32(3)).reshape(-1)[:length].astype(np.uint8)


def quantize(residual: np.ndarray, grad: np.ndarray, alpha: float):
    """Threshold-quantize r+g with error feedback — codec.py:164-194.

    Returns ``(words, new_residual)``; the input residual is NOT modified (the
    reference mutates in place, codec.py:192 — callers here keep the returned
    array). Raises OracleNumericError(first non-finite index) before producing
    anything (codec.py:181-185).
    """
    if alpha <= 0:
        raise ValueError("threshold alpha must be > 0")
    g = np.asarray(grad, dtype=np.float64)                       # codec.py:176
    r = np.asarray(residual, dtype=np.float64)
    if g.shape != r.shape:
        raise ValueError("gradient length does not match residual")
    acc = r + g                                                  # codec.py:181
    finite = np.isfinite(acc)
    if not finite.all():                                         # codec.py:182-185
        bad = int(np.argmin(finite))
        raise OracleNumericError(f"non-finite accumulated gradient at element {bad}", bad)
    plus = acc >= alpha                                          # codec.py:186
    minus = acc <= -alpha                                        # codec.py:187
    sym = np.zeros(acc.shape[0], dtype=np.uint8)
    sym[plus] = SYM_PLUS
    sym[minus] = SYM_MINUS
    emitted = np.where(plus, alpha, 0.0) + np.where(minus, -alpha, 0.0)  # codec.py:191
    return pack_symbols(sym), acc - emitted                      # codec.py:192-193


def quantize_f32(residual: np.ndarray, grad: np.ndarray, alpha: float):
    """FAST-MODE restatement of codec.py:181-193 in float32 (NOT the reference's arithmetic,
    which is fp64): the same operations in the same order with fp32 operands and threshold
    a = float32(alpha) — acc = r + g; plus = acc >= a; minus = acc <= -a; emitted =
    where(plus, a, 0) + where(minus, -a, 0); r' = acc - emitted. Pins the GPU's fp32-residual
    mode (cdsgd_quantize_f32r) bitwise; same error semantics as quantize()."""
    if alpha <= 0:
        raise ValueError("threshold alpha must be > 0")
    a = np.float32(alpha)
    g = np.asarray(grad, dtype=np.float32)
    r = np.asarray(residual, dtype=np.float32)
    if g.shape != r.shape:
        raise ValueError("gradient length does not match residual")
    acc = r + g                                                  # codec.py:181, fp32
    finite = np.isfinite(acc)
    if not finite.all():                                         # codec.py:182-185
        bad = int(np.argmin(finite))
        raise OracleNumericError(f"non-finite accumulated gradient at element {bad}", bad)
    plus = acc >= a                                              # codec.py:186
    minus = acc <= -a                                            # codec.py:187
    sym = np.zeros(acc.shape[0], dtype=np.uint8)
    sym[plus] = SYM_PLUS
    sym[minus] = SYM_MINUS
    emitted = np.where(plus, a, np.float32(0)) + np.where(minus, -a, np.float32(0))  # codec.py:191, fp32
    return pack_symbols(sym), (acc - emitted).astype(np.float32)  # codec.py:192-193


def quantize_layout_f32(residual, grad, alpha, sizes):
    """quantize_layout with the fp32 restatement (fast mode)."""
    eoff, woff = layout_offsets(sizes)
    words = np.zeros(int(woff[-1]), dtype=np.uint32)
    r_new = np.empty(int(eoff[-1]), dtype=np.float32)
    for k in range(len(sizes)):
        sl = slice(int(eoff[k]), int(eoff[k + 1]))
        try:
            w, r = quantize_f32(residual[sl], grad[sl], alpha)
        except OracleNumericError as exc:
            exc.key = k
            raise
        words[int(woff[k]) : int(woff[k + 1])] = w
        r_new[sl] = r
    return words, r_new


def dequantize(words: np.ndarray, threshold: float, length: int) -> np.ndarray:
    """Decode to {-t, 0, +t} float64; reserved 11 -> error at first index — codec.py:197-206."""
    sym = unpack_symbols(words, length)
    if (sym > SYM_MINUS).any():
        bad = int(np.argmax(sym > SYM_MINUS))
        raise OracleCorruptPayload(f"reserved symbol 11 at element {bad}")
    out = np.zeros(length, dtype=np.float64)
    out[sym == SYM_PLUS] = threshold
    out[sym == SYM_MINUS] = -threshold
    return out


def payload_to_bytes(words: np.ndarray, threshold: float, length: int) -> bytes:
    """13-byte <BdI header + LE u32 words — codec.py:90-93."""
    return _HEADER.pack(CODEC_TAG, threshold, length) + np.asarray(words, "<u4").tobytes()


def payload_from_bytes(data: bytes):
    """codec.py:95-108."""
    if len(data) < PAYLOAD_HEADER_BYTES:
        raise OracleCorruptPayload("payload shorter than its header")
    tag, threshold, length = _HEADER.unpack_from(data)
    if tag != CODEC_TAG:
        raise OracleCorruptPayload(f"unknown codec tag 0x{tag:02X}")
    body = data[PAYLOAD_HEADER_BYTES:]
    if len(body) != 4 * words_needed(length):
        raise OracleCorruptPayload("payload body size mismatch")
    return np.frombuffer(body, dtype="<u4").astype(np.uint32), threshold, length


# ----------------------------------------------------------------------------- layout


def layout_offsets(sizes):
    """Key element offsets and packed-word offsets (numcore.py:48-84; codec.py:49-50).

    Packing restarts at every key because the reference quantizes each key
    slice separately (engine.py:397-402)."""
    sizes = [int(s) for s in sizes]
    if not sizes or min(sizes) < 1:
        raise ValueError("layout needs keys of length >= 1")
    eoff = np.zeros(len(sizes) + 1, dtype=np.int64)
    woff = np.zeros(len(sizes) + 1, dtype=np.int64)
    eoff[1:] = np.cumsum(sizes)
    woff[1:] = np.cumsum([words_needed(s) for s in sizes])
    return eoff, woff


def quantize_layout(residual, grad, alpha, sizes):
    """Per-key quantize over a flat layout -> (flat words, new residual) (engine.py:397-402).

    Raises OracleNumericError with ``.key`` and the key-local ``.index``."""
    eoff, woff = layout_offsets(sizes)
    words = np.zeros(int(woff[-1]), dtype=np.uint32)
    r_new = np.empty(int(eoff[-1]), dtype=np.float64)
    for k in range(len(sizes)):
        sl = slice(int(eoff[k]), int(eoff[k + 1]))
        try:
            w, r = quantize(residual[sl], grad[sl], alpha)
        except OracleNumericError as exc:
            exc.key = k
            raise
        words[int(woff[k]) : int(woff[k + 1])] = w
        r_new[sl] = r
    return words, r_new


def dequantize_layout(words, alpha, sizes):
    eoff, woff = layout_offsets(sizes)
    out = np.empty(int(eoff[-1]), dtype=np.float64)
    for k, n in enumerate(sizes):
        out[int(eoff[k]) : int(eoff[k + 1])] = dequantize(
            words[int(woff[k]) : int(woff[k + 1])], alpha, int(n)
        )
    return out


# ----------------------------------------------------------------------------- engine rules


def should_compress(count: int, k: int) -> bool:
    """engine.py:217-223."""
    if k < 1 or count < 1:
        raise ValueError("k and count must be >= 1")
    return count % k != 0


def server_aggregate(vectors) -> np.ndarray:
    """Ascending-worker-id sum of decoded/full vectors, then /N — engine.py:249-255.

    ``vectors`` is the list of already-decoded float64 vectors in worker order."""
    total = None
    for v in vectors:
        v = np.asarray(v, dtype=np.float64)
        total = v.copy() if total is None else total + v
    return total / len(vectors)


def global_update(weights: np.ndarray, mean: np.ndarray, eta: float) -> np.ndarray:
    """W <- W - eta*mean, per key (identical elementwise) — engine.py:258-265, 511."""
    weights -= eta * mean
    return weights


def local_update(base: np.ndarray, grad: np.ndarray, eta_l: float) -> np.ndarray:
    """base - eta_l*grad (new vector) — engine.py:268-274."""
    return base - eta_l * np.asarray(grad, dtype=np.float64)


# ----------------------------------------------------------------------------- synthetic inputs


def synthetic_grad(seed: int, t: int, w: int, n: int, scale: float = 0.3) -> np.ndarray:
    """g_{t,w} = scale*N(0,1) as float32 from default_rng([seed, t, w])."""
    rng = np.random.default_rng([seed, t, w])
    return (scale * rng.standard_normal(n)).astype(np.float32)


def synthetic_weights(seed: int, n: int) -> np.ndarray:
    """W_0 = N(0,1) float32 from default_rng([seed, 999])."""
    return np.random.default_rng([seed, 999]).standard_normal(n).astype(np.float32)


# ----------------------------------------------------------------------------- lock-step engine


@dataclass
class OracleHP:
    """Subset of engine.HyperParams (engine.py:96-144) the hot path reads."""

    algo: str = "cdsgd"
    workers: int = 1
    eta_global: float = 0.1
    eta_local: float | None = None
    k: int = 5
    alpha: float = 0.5
    warmup_n: int = 5
    force_compress: bool = False
    bypass_local: bool = False

    @property
    def local_lr(self) -> float:
        return self.eta_global if self.eta_local is None else self.eta_local


@dataclass
class _OWorker:
    wid: int
    t: int = 0
    current_global: np.ndarray = None
    slots: list = field(default_factory=lambda: [None, None])
    residual: np.ndarray = None


class LockstepOracle:
    """Restatement of Worker/ServerNode/_run_lockstep (engine.py:288-663) for
    synthetic gradients: the gradient fed at (t, w) replaces ``loss_and_grad``
    (engine.py:363); everything else — warm-up, parity slots, should_compress,
    per-key quantize, ascending-wid aggregation, server apply, pull — follows the
    reference line for line, in float64.
    """

    def __init__(self, w0: np.ndarray, sizes, hp: OracleHP, residual: str = "f64"):
        """residual="f32": the fast-mode restatement (quantize_f32); everything else fp64."""
        self.hp = hp
        self.residual_dtype = residual
        self.sizes = [int(s) for s in sizes]
        self.n = int(sum(self.sizes))
        self.W = np.asarray(w0, dtype=np.float64).copy()          # ServerNode.weights, engine.py:448
        self.uses_local = hp.algo in ("lusgd", "cdsgd") and not hp.bypass_local   # engine.py:310
        self.quantizes = hp.algo in ("bitsgd", "cdsgd")           # engine.py:312
        self.n_warmup = hp.warmup_n if hp.algo in ("lusgd", "cdsgd") else 0       # engine.py:314
        self.workers = []
        for w in range(hp.workers):
            ow = _OWorker(w, 0, self.W.copy(), [None, None],
                          np.zeros(self.n, dtype=np.float32 if residual == "f32" else np.float64))
            if self.uses_local and self.n_warmup == 0:           # engine.py:318-322
                ow.slots = [self.W.copy(), self.W.copy()]
            self.workers.append(ow)
        self.t = 0
        self.weights_after: list[np.ndarray] = []
        self.compressed: list[bool] = []
        self.grad_norms: list[float] = []
        self.words: dict[tuple[int, int], np.ndarray] = {}

    def _in_warmup(self, w: _OWorker) -> bool:                   # engine.py:332-333
        return self.uses_local and w.t < self.n_warmup

    def compute_weights(self, w: int) -> np.ndarray:
        """Weights worker w computes its next gradient at — engine.py:335-343."""
        ow = self.workers[w]
        if self.uses_local and not self._in_warmup(ow):
            if ow.slots[ow.t % 2] is None:
                raise RuntimeError("local slot never written")
            return ow.slots[ow.t % 2]
        return ow.current_global

    def _push_compressed(self, ow: _OWorker) -> bool:            # engine.py:345-355
        if self._in_warmup(ow):
            return False
        if self.hp.algo == "bitsgd":
            return True
        if self.hp.algo == "cdsgd":
            if self.hp.force_compress:
                return True
            return should_compress(ow.t - self.n_warmup + 1, self.hp.k)
        return False

    def step(self, grads) -> None:
        """One lock-step round: every worker computes+pushes, server commits, all pull."""
        hp = self.hp
        contrib = []
        flags = set()
        for ow, g in zip(self.workers, grads):                    # engine.py:627-632
            t = ow.t
            weights = self.compute_weights(ow.wid)
            g64 = np.asarray(g, dtype=np.float64)
            if self.uses_local:                                   # engine.py:373-392
                if self._in_warmup(ow):
                    if t == self.n_warmup - 1:
                        slot = self.n_warmup % 2
                        base = ow.slots[slot] if ow.slots[slot] is not None else weights
                        ow.slots[slot] = local_update(base, g64, hp.local_lr)
                else:
                    pending = (t + 1) % 2
                    ow.slots[pending] = local_update(ow.slots[pending], g64, hp.local_lr)
            compressed = self._push_compressed(ow)               # engine.py:394
            flags.add(compressed)
            if compressed:                                        # engine.py:397-404
                if self.residual_dtype == "f32":
                    words, ow.residual = quantize_layout_f32(ow.residual, np.asarray(g, np.float32), hp.alpha,
                                                             self.sizes)
                else:
                    words, ow.residual = quantize_layout(ow.residual, g64, hp.alpha, self.sizes)
                self.words[(t, ow.wid)] = words
                contrib.append(dequantize_layout(words, hp.alpha, self.sizes))
            else:
                contrib.append(g64.copy())                        # engine.py:406
        assert len(flags) == 1, "workers disagree on compression"
        mean = server_aggregate(contrib)                          # engine.py:510 (all keys)
        self.W -= hp.eta_global * mean                            # engine.py:511
        self.grad_norms.append(float(np.linalg.norm(mean)))       # engine.py:521
        self.weights_after.append(self.W.copy())                  # engine.py:524
        self.compressed.append(flags.pop())
        for ow in self.workers:                                   # engine.py:410-430
            t = ow.t
            pulled = self.W.copy()
            ow.current_global = pulled
            if self.uses_local:
                if self._in_warmup(ow):
                    if t == self.n_warmup - 2:
                        ow.slots[self.n_warmup % 2] = pulled.copy()
                    if t == self.n_warmup - 1:
                        ow.slots[(self.n_warmup + 1) % 2] = pulled.copy()
                else:
                    ow.slots[t % 2] = pulled.copy()
            ow.t += 1
        self.t += 1
