"""Ternary 2-bit gradient codec with residual error feedback — B200 edition.

Drop-in for the reference ``cdsgd.codec`` (pkg/src/cdsgd/codec.py): same names,
argument meaning, error classes and bit layout (symbol j -> bits 2(j%16)..+1 of
u32 word j//16, LE; 00 zero, 01 +alpha, 10 -alpha, 11 invalid), but vectors
are CUDA tensors and every vector operation is a kernel of libcdsgd_b200.so.
NumPy inputs are accepted and uploaded; outputs stay on the device.

Differences that are representation-only:
  * ``ResidualState`` keeps two fp64 buffers and swaps them on success, so the
    quantizer reads the old residual and writes the new one in a single pass
    while keeping the reference's no-mutation-on-error guarantee
    (codec.py:181-185). ``state.residual`` always returns the live buffer.
  * ``quantize_keys`` quantizes every key of a Layout in ONE launch, the way
    Worker.compute_push loops over keys (engine.py:397-402).
"""

from __future__ import annotations

import struct
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .layout import Layout

SYM_ZERO = 0
SYM_PLUS = 1
SYM_MINUS = 2
SYMBOLS_PER_WORD = 16
CODEC_TAG = 0x02
_HEADER = struct.Struct("<BdI")
PAYLOAD_HEADER_BYTES = _HEADER.size  # 13


class CorruptPayloadError(ValueError):
    """Payload failed validation (reserved symbol, bad tag, bad sizes) — codec.py:33-34."""


class CodecError(ValueError):
    """Invalid codec arguments — codec.py:37-38."""


class CodecNumericError(ArithmeticError):
    """Non-finite value fed into the quantizer; carries the element index — codec.py:41-46.

    ``index`` is local to the key slice (as in the reference, which quantizes per
    key); ``key`` names that key and ``round`` the engine round when known."""

    def __init__(self, message: str, index: int, key: int = 0, round: int | None = None):
        super().__init__(message)
        self.index = index
        self.key = key
        self.round = round


def _words_needed(n: int) -> int:
    return (n + SYMBOLS_PER_WORD - 1) // SYMBOLS_PER_WORD


def payload_bytes(n_elements: int) -> int:
    """Packed-code size in bytes: 4 * ceil(n/16) (codec.py:53-57)."""
    if n_elements < 0:
        raise CodecError("element count must be >= 0")
    return 4 * _words_needed(n_elements)


def compression_ratio(n_elements: int) -> float:
    """Packed size vs a 4-byte-per-element baseline (codec.py:60-64)."""
    if n_elements == 0:
        return 1.0
    return (4.0 * n_elements) / payload_bytes(n_elements)


def serialized_payload_bytes(n_elements: int) -> int:
    """13-byte header plus the packed words (codec.py:67-69)."""
    return PAYLOAD_HEADER_BYTES + payload_bytes(n_elements)


# ----------------------------------------------------------------------------- helpers


def _require_cuda():
    if not torch.cuda.is_available():
        raise _lib.LibraryError("CUDA device required: the CD-SGD codec runs only on the GPU (no CPU fallback)")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _device_tensor(x, dtype=None) -> torch.Tensor:
    _require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.cuda()
    return t.contiguous()


_SINGLE: dict[int, Layout] = {}


def _single_layout(n: int) -> Layout:
    lay = _SINGLE.get(n)
    if lay is None:
        if len(_SINGLE) > 256:
            _SINGLE.clear()
        lay = _SINGLE[n] = Layout([("w", n)])
    return lay


class _ErrWord:
    """Per-device 2-word device error slot (CDSGD_NO_ERROR = all ones)."""

    _cache: dict[int, torch.Tensor] = {}

    @classmethod
    def fresh(cls) -> torch.Tensor:
        dev = torch.cuda.current_device()
        t = cls._cache.get(dev)
        if t is None:
            t = cls._cache[dev] = torch.empty(2, dtype=torch.int64, device=f"cuda:{dev}")
        t.fill_(-1)
        return t

    @staticmethod
    def read(t: torch.Tensor) -> list[int]:
        return [int(v) & 0xFFFFFFFFFFFFFFFF for v in t.cpu().tolist()]


def _locate(layout: Layout, flat: int) -> tuple[int, int]:
    for span in layout.spans:
        if span.start <= flat < span.start + span.length:
            return span.key, flat - span.start
    raise IndexError(flat)


# ----------------------------------------------------------------------------- types


class QuantizedPayload:
    """Packed 2-bit symbols with their threshold and element count (codec.py:72-120)."""

    def __init__(self, words, threshold: float, length: int):
        if isinstance(words, torch.Tensor):
            w = words
            if w.dtype != torch.uint32:
                w = w.view(torch.uint32) if w.dtype == torch.int32 else w.to(torch.int64).to(torch.uint32)
        else:
            w = torch.from_numpy(np.ascontiguousarray(np.asarray(words, dtype=np.uint32)))
        self.words = w.contiguous() if w.dim() == 1 else w.reshape(-1)
        self.threshold = float(threshold)
        self.length = int(length)
        if self.threshold <= 0:
            raise CorruptPayloadError("threshold must be > 0")
        if self.length < 0 or self.words.shape[0] != _words_needed(self.length):
            raise CorruptPayloadError(
                f"expected {_words_needed(self.length)} words for {self.length} elements, "
                f"got {self.words.shape[0]}"
            )

    def to_bytes(self) -> bytes:
        body = self.words.cpu().numpy().astype("<u4").tobytes()
        return _HEADER.pack(CODEC_TAG, self.threshold, self.length) + body

    @classmethod
    def from_bytes(cls, data: bytes, device=None) -> "QuantizedPayload":
        if len(data) < PAYLOAD_HEADER_BYTES:
            raise CorruptPayloadError("payload shorter than its header")
        tag, threshold, length = _HEADER.unpack_from(data)
        if tag != CODEC_TAG:
            raise CorruptPayloadError(f"unknown codec tag 0x{tag:02X}")
        body = data[PAYLOAD_HEADER_BYTES:]
        if len(body) != 4 * _words_needed(length):
            raise CorruptPayloadError(
                f"payload body is {len(body)} bytes, expected {4 * _words_needed(length)}"
            )
        words = torch.from_numpy(np.frombuffer(body, dtype="<u4").astype(np.uint32))
        if device is not None or torch.cuda.is_available():
            words = words.to(device if device is not None else "cuda")
        return cls(words, threshold, length)

    @property
    def nbytes(self) -> int:
        return serialized_payload_bytes(self.length)

    def __eq__(self, other) -> bool:
        return (
            isinstance(other, QuantizedPayload)
            and self.threshold == other.threshold
            and self.length == other.length
            and torch.equal(self.words.cpu(), other.words.cpu())
        )

    def __repr__(self) -> str:
        return f"QuantizedPayload(length={self.length}, threshold={self.threshold}, words={self.words.shape[0]})"


class ResidualState:
    """Per-(worker, key) fp64 accumulator of not-yet-emitted gradient mass (codec.py:123-137)."""

    def __init__(self, residual, owner: tuple[int, int] = (0, 0)):
        t = _device_tensor(residual, torch.float64)
        if t.dim() != 1:
            raise CodecError("residual must be a 1-D vector")
        if isinstance(residual, torch.Tensor) and t.data_ptr() == residual.data_ptr():
            t = t.clone()  # own the buffer, like np.ascontiguousarray copies a foreign dtype
        self._bufs = [t, None]
        self._cur = 0
        self.owner = tuple(owner)

    @classmethod
    def zeros(cls, length: int, owner: tuple[int, int] = (0, 0), device=None) -> "ResidualState":
        _require_cuda()
        return cls(torch.zeros(length, dtype=torch.float64, device=device or "cuda"), owner)

    @property
    def residual(self) -> torch.Tensor:
        return self._bufs[self._cur]

    @residual.setter
    def residual(self, value) -> None:
        self._bufs = [_device_tensor(value, torch.float64).clone(), None]
        self._cur = 0

    def _spare(self) -> torch.Tensor:
        s = self._bufs[self._cur ^ 1]
        cur = self._bufs[self._cur]
        if s is None or s.shape != cur.shape or s.device != cur.device:
            s = torch.empty_like(cur)
            self._bufs[self._cur ^ 1] = s
        return s

    def _commit(self) -> None:
        self._cur ^= 1


# ----------------------------------------------------------------------------- operations


def pack_symbols(symbols) -> torch.Tensor:
    """Pack ternary symbols into uint32 words, 16 two-bit codes per word (codec.py:140-151)."""
    s = _device_tensor(symbols)
    if s.dtype != torch.uint8:
        if s.numel() and (int(s.min()) < 0 or int(s.max()) > 255):
            raise CorruptPayloadError("symbols must be in {0, 1, 2}")
        s = s.to(torch.uint8)
    n = s.shape[0]
    words = torch.empty(_words_needed(n), dtype=torch.uint32, device=s.device)
    if n == 0:
        return words
    err = _ErrWord.fresh()
    _lib.check(_lib.lib().cdsgd_pack_symbols(s.data_ptr(), n, words.data_ptr(), err.data_ptr(), _stream()),
               "pack_symbols")
    if _ErrWord.read(err)[0] != _lib.NO_ERROR:
        raise CorruptPayloadError("symbols must be in {0, 1, 2}")
    return words


def unpack_symbols(words, length: int) -> torch.Tensor:
    """Exact inverse of pack_symbols for the first `length` symbols (codec.py:154-161)."""
    w = _device_tensor(words)
    if w.dtype != torch.uint32:
        w = w.view(torch.uint32) if w.dtype == torch.int32 else w.to(torch.int64).to(torch.uint32)
    if length < 0 or length > w.shape[0] * SYMBOLS_PER_WORD:
        raise CodecError(f"{length} symbols do not fit in {w.shape[0]} words")
    out = torch.empty(length, dtype=torch.uint8, device=w.device)
    if length:
        _lib.check(_lib.lib().cdsgd_unpack_symbols(w.data_ptr(), length, out.data_ptr(), _stream()),
                   "unpack_symbols")
    return out


def _grad_dtype(g: torch.Tensor) -> int:
    if g.dtype == torch.float32:
        return _lib.F32
    if g.dtype == torch.float64:
        return _lib.F64
    raise CodecError(f"gradient dtype {g.dtype} not supported (float32 or float64)")


def quantize(residual: ResidualState, grad, alpha: float) -> tuple[QuantizedPayload, ResidualState]:
    """Threshold-quantize residual + grad; the leftover stays in the residual (codec.py:164-194).

    Per element, a = r + g (fp64): +alpha if a >= alpha, -alpha if a <= -alpha,
    else zero; the new residual is a minus the emitted value. The state is updated
    and returned with the payload; on a non-finite accumulator CodecNumericError
    (first index) is raised and the state is left untouched.
    """
    if alpha <= 0:
        raise CodecError("threshold alpha must be > 0")
    g = _device_tensor(grad)
    if g.dtype not in (torch.float32, torch.float64):
        g = g.to(torch.float64)
    r = residual.residual
    if tuple(g.shape) != tuple(r.shape):
        raise CodecError(f"gradient length {tuple(g.shape)} does not match residual {tuple(r.shape)}")
    n = r.shape[0]
    if n == 0:
        return QuantizedPayload(torch.empty(0, dtype=torch.uint32, device=r.device), float(alpha), 0), residual
    lay = _single_layout(n)
    words = torch.empty(_words_needed(n), dtype=torch.uint32, device=r.device)
    out = residual._spare()
    err = _ErrWord.fresh()
    _lib.check(
        _lib.lib().cdsgd_quantize(lay.handle().ptr, g.data_ptr(), _grad_dtype(g), r.data_ptr(), out.data_ptr(),
                                  words.data_ptr(), float(alpha), err.data_ptr(), 0, _stream()),
        "quantize",
    )
    bad = _ErrWord.read(err)[0]
    if bad != _lib.NO_ERROR:
        raise CodecNumericError(f"non-finite accumulated gradient at element {bad}", bad)
    residual._commit()
    return QuantizedPayload(words, float(alpha), n), residual


def quantize_keys(
    residual: ResidualState, grad, alpha: float, layout: Layout
) -> tuple[list[QuantizedPayload], torch.Tensor, ResidualState]:
    """Quantize every key of `layout` in one launch (engine.py:397-402 loop, fused).

    Returns (per-key payloads as views of one packed buffer, the packed buffer,
    the updated state). On a non-finite value raises CodecNumericError with the
    key and key-local index of the first offender; the state is untouched."""
    if alpha <= 0:
        raise CodecError("threshold alpha must be > 0")
    g = _device_tensor(grad)
    r = residual.residual
    if g.shape[0] != layout.total or r.shape[0] != layout.total:
        raise CodecError("gradient/residual length does not match the layout")
    words = torch.empty(layout.n_words, dtype=torch.uint32, device=r.device)
    out = residual._spare()
    err = _ErrWord.fresh()
    _lib.check(
        _lib.lib().cdsgd_quantize(layout.handle().ptr, g.data_ptr(), _grad_dtype(g), r.data_ptr(),
                                  out.data_ptr(), words.data_ptr(), float(alpha), err.data_ptr(), 0, _stream()),
        "quantize_keys",
    )
    bad = _ErrWord.read(err)[0]
    if bad != _lib.NO_ERROR:
        key, idx = _locate(layout, bad)
        raise CodecNumericError(f"non-finite accumulated gradient at element {idx}", idx, key=key)
    residual._commit()
    payloads = []
    w0 = 0
    for span in layout.spans:
        nw = _words_needed(span.length)
        payloads.append(QuantizedPayload(words[w0 : w0 + nw], float(alpha), span.length))
        w0 += nw
    return payloads, words, residual


def dequantize(payload: QuantizedPayload) -> torch.Tensor:
    """Decode a payload to float64 values in {-threshold, 0, +threshold} (codec.py:197-206)."""
    n = payload.length
    w = _device_tensor(payload.words)
    out = torch.empty(n, dtype=torch.float64, device=w.device)
    if n == 0:
        return out
    err = _ErrWord.fresh()
    _lib.check(
        _lib.lib().cdsgd_dequantize_sum(_single_layout(n).handle().ptr, w.data_ptr(), 1, w.shape[0],
                                        payload.threshold, out.data_ptr(), err.data_ptr(), _stream()),
        "dequantize",
    )
    bad = _ErrWord.read(err)[0]
    if bad != _lib.NO_ERROR:
        raise CorruptPayloadError(f"reserved symbol 11 at element {bad}")
    return out


def dequantize_sum(payloads: Sequence[QuantizedPayload]) -> torch.Tensor:
    """Ascending-order decode-sum / len(payloads) in fp64 (engine.py:249-255, quantized branch).

    Every payload is decoded with its OWN threshold, as the reference does (dequantize per
    contribution, engine.py:251): equal thresholds take the single fused kernel, mixed ones
    decode payload by payload and add in ascending order (the same fp64 operations).
    Payloads of different lengths cannot be summed (the reference server rejects them,
    engine.py:500-504): CodecError."""
    if not payloads:
        raise CodecError("need at least one payload")
    n = payloads[0].length
    if any(p.length != n for p in payloads):
        raise CodecError(f"payload lengths differ: {[p.length for p in payloads]}")
    thr = payloads[0].threshold
    if any(p.threshold != thr for p in payloads):
        total = None
        for p in payloads:
            d = dequantize(p)
            total = d if total is None else total + d
        return total / len(payloads)
    stacked = torch.stack([_device_tensor(p.words).view(torch.int32) for p in payloads]).view(torch.uint32)
    out = torch.empty(n, dtype=torch.float64, device=stacked.device)
    if n == 0:
        return out
    err = _ErrWord.fresh()
    _lib.check(
        _lib.lib().cdsgd_dequantize_sum(_single_layout(n).handle().ptr, stacked.data_ptr(), len(payloads),
                                        stacked.shape[1], thr, out.data_ptr(), err.data_ptr(), _stream()),
        "dequantize_sum",
    )
    bad = _ErrWord.read(err)[0]
    if bad != _lib.NO_ERROR:
        raise CorruptPayloadError(f"reserved symbol 11 at element {bad}")
    return out
