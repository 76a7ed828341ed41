"""Wire-format interop with the reference parameter server.

Byte-exact encoder/decoder of the reference's frames (pkg/src/cdsgd/protocol.py:29-171):
a 20-byte little-endian header ``<HBBHHQI`` = magic 0xCD5D, version 1, variant,
worker, key, iteration, payload length, followed by the payload — a serialized
``QuantizedPayload`` (13-byte ``<BdI`` header + LE u32 words, codec.py:90-108) for
compressed pushes, raw LE float64 values for full pushes and weight replies.

With it a GPU worker can push the codes its K1/fused kernel produced to the unmodified
reference ``ServerNode`` (socket transport, engine.py:666-727) and consume its weight
replies; ``CDSGDWorker.round_payloads(t)`` exposes the per-key payloads of a round.
This is host-side framing (a device->host copy of the packed words), not the hot path.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from .codec import QuantizedPayload

MAGIC = 0xCD5D
VERSION = 1
_HEADER = struct.Struct("<HBBHHQI")
HEADER_BYTES = _HEADER.size  # 20 (SPEC.md:201 says 18; the code is authoritative)

VARIANT_PUSH_FULL = 1
VARIANT_PUSH_QUANTIZED = 2
VARIANT_PULL_REQUEST = 3
VARIANT_WEIGHTS = 4
VARIANT_SHUTDOWN = 5


class ProtocolError(ValueError):
    """Frame failed validation (bad magic, version, or variant) — protocol.py:42-43."""


class FramingError(ProtocolError):
    """Frame shorter than its declared size — protocol.py:46-47."""


@dataclass
class Frame:
    variant: int
    worker: int
    key: int
    iteration: int
    payload: object = None  # QuantizedPayload | np.ndarray (float64) | None


def _f64_bytes(values) -> bytes:
    if isinstance(values, torch.Tensor):
        values = values.detach().to("cpu", torch.float64).numpy()
    return np.ascontiguousarray(values, dtype="<f8").tobytes()


def _frame(variant: int, worker: int, key: int, iteration: int, body: bytes) -> bytes:
    try:
        header = _HEADER.pack(MAGIC, VERSION, variant, worker, key, iteration, len(body))
    except struct.error as exc:
        raise ProtocolError(f"field out of range for the wire format: {exc}") from exc
    return header + body


def encode_push_quantized(worker: int, iteration: int, key: int, payload: QuantizedPayload) -> bytes:
    """PushQuantized frame (protocol.py:123-125)."""
    return _frame(VARIANT_PUSH_QUANTIZED, worker, key, iteration, payload.to_bytes())


def encode_push_full(worker: int, iteration: int, key: int, values) -> bytes:
    """PushFull frame: values as LE float64 (protocol.py:120-122)."""
    return _frame(VARIANT_PUSH_FULL, worker, key, iteration, _f64_bytes(values))


def encode_pull_request(worker: int, iteration: int) -> bytes:
    return _frame(VARIANT_PULL_REQUEST, worker, 0, iteration, b"")


def encode_weights(iteration: int, key: int, values) -> bytes:
    return _frame(VARIANT_WEIGHTS, 0, key, iteration, _f64_bytes(values))


def encode_shutdown() -> bytes:
    return _frame(VARIANT_SHUTDOWN, 0, 0, 0, b"")


def decode_frame(data: bytes, device=None) -> Frame:
    """Exact inverse of the encoders (protocol.py:143-171), same errors."""
    if len(data) < HEADER_BYTES:
        raise FramingError(f"frame is {len(data)} bytes, header needs {HEADER_BYTES}")
    magic, version, variant, worker, key, iteration, payload_len = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise ProtocolError(f"bad magic 0x{magic:04X}")
    if version != VERSION:
        raise ProtocolError(f"unsupported version {version}")
    body = data[HEADER_BYTES:]
    if len(body) != payload_len:
        raise FramingError(f"declared payload {payload_len} bytes, got {len(body)}")
    if variant in (VARIANT_PUSH_FULL, VARIANT_WEIGHTS):
        if payload_len % 8:
            raise FramingError("payload must be whole float64 values")
        values = np.frombuffer(body, dtype="<f8").astype(np.float64)
        if variant == VARIANT_WEIGHTS:
            return Frame(variant, 0, key, iteration, values)
        return Frame(variant, worker, key, iteration, values)
    if variant == VARIANT_PUSH_QUANTIZED:
        return Frame(variant, worker, key, iteration, QuantizedPayload.from_bytes(body, device=device))
    if variant == VARIANT_PULL_REQUEST:
        return Frame(variant, worker, 0, iteration)
    if variant == VARIANT_SHUTDOWN:
        return Frame(variant, 0, 0, 0)
    raise ProtocolError(f"unknown variant tag {variant}")


def round_frames(worker_id: int, iteration: int, payloads=None, grad=None, layout=None) -> list[bytes]:
    """The frames Worker.compute_push sends for one round (engine.py:397-407), one per key:
    PushQuantized from per-key payloads, or PushFull slices of `grad` over `layout`."""
    if payloads is not None:
        return [encode_push_quantized(worker_id, iteration, k, p) for k, p in enumerate(payloads)]
    if grad is None or layout is None:
        raise ValueError("need payloads, or grad and layout")
    g = grad.detach().to("cpu", torch.float64).numpy() if isinstance(grad, torch.Tensor) else np.asarray(grad)
    return [encode_push_full(worker_id, iteration, s.key, g[s.start:s.start + s.length]) for s in layout.spans]
