"""Update rules of CD-SGD on the GPU — drop-in for the reference ``cdsgd.engine`` hot path.

Same names, argument meaning and errors as pkg/src/cdsgd/engine.py:96-144, 217-274:
``HyperParams``, ``should_compress``, ``server_aggregate``, ``global_update``,
``local_update``, plus ``KeyedVector`` (numcore.py:87-115) holding a CUDA tensor.
Vector work runs in libcdsgd_b200.so kernels; the per-round choreography
(Worker/ServerNode, engine.py:288-558) is the native step engine driven by
``paper_2106_10796_b200.worker.CDSGDWorker``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .codec import QuantizedPayload, _device_tensor, _stream, dequantize_sum
from .layout import Layout, LayoutError

ALGORITHMS = ("ssgd", "lusgd", "bitsgd", "cdsgd")


class ConfigError(ValueError):
    """Invalid model, dataset, or hyperparameter configuration (numcore.py:24-25)."""


class ProtocolViolation(RuntimeError):
    """The synchronous push/pull contract was broken (engine.py:81-82)."""


class SchedulingError(RuntimeError):
    """A worker needed state that its pull had not produced yet (engine.py:85-86)."""


@dataclass
class HyperParams:
    """Training configuration (engine.py:96-144); eta_local defaults to eta_global."""

    algo: str
    workers: int = 1
    eta_global: float = 0.1
    eta_local: Optional[float] = None
    k: int = 5
    alpha: float = 0.5
    warmup_n: int = 5
    batch_size: int = 32
    epochs: int = 1
    iters: Optional[int] = None
    seed: int = 0

    def validate(self) -> "HyperParams":
        if self.algo not in ALGORITHMS:
            raise ConfigError(f"algo must be one of {', '.join(ALGORITHMS)}; got {self.algo!r}")
        if self.workers < 1:
            raise ConfigError("workers must be ≥ 1")
        if self.eta_global <= 0:
            raise ConfigError("eta_global must be > 0")
        if self.eta_local is not None and self.eta_local <= 0:
            raise ConfigError("eta_local must be > 0")
        if self.k < 1:
            raise ConfigError("k must be ≥ 1")
        if self.alpha <= 0:
            raise ConfigError("alpha must be > 0")
        if self.warmup_n < 0:
            raise ConfigError("warmup_n must be ≥ 0")
        if self.batch_size < 1:
            raise ConfigError("batch_size must be ≥ 1")
        if self.iters is None and self.epochs < 1:
            raise ConfigError("epochs must be ≥ 1")
        if self.iters is not None and self.iters < 1:
            raise ConfigError("iters must be ≥ 1")
        return self

    @property
    def local_lr(self) -> float:
        return self.eta_global if self.eta_local is None else self.eta_local


class KeyedVector:
    """Flat vector plus the key layout that partitions it (numcore.py:87-115).

    ``values`` is a 1-D CUDA tensor (fp32 or fp64); NumPy input is uploaded as fp64
    like the reference's ``np.ascontiguousarray(values, dtype=np.float64)``."""

    def __init__(self, values, layout: Layout):
        if isinstance(values, torch.Tensor):
            t = _device_tensor(values)
            if t.dtype not in (torch.float32, torch.float64):
                t = t.to(torch.float64)
        else:
            t = _device_tensor(np.asarray(values, dtype=np.float64))
        if t.dim() != 1 or t.shape[0] != layout.total:
            raise LayoutError(f"vector length {tuple(t.shape)} does not match layout total {layout.total}")
        self.values = t
        self.layout = layout

    def copy(self) -> "KeyedVector":
        return KeyedVector(self.values.clone(), self.layout)

    def key(self, key: int) -> torch.Tensor:
        return self.values[self.layout.slice(key)]

    def same_layout(self, other: "KeyedVector") -> bool:
        return self.layout == other.layout


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.F32
    if t.dtype == torch.float64:
        return _lib.F64
    raise ConfigError(f"unsupported dtype {t.dtype}")


def should_compress(count: int, k: int) -> bool:
    """True on the k-1 compressing iterations of each period: count % k != 0 (engine.py:217-223)."""
    if k < 1:
        raise ConfigError("k must be ≥ 1")
    if count < 1:
        raise ConfigError("count must be ≥ 1")
    return count % k != 0


def server_aggregate(
    contributions: dict[int, tuple[str, object]],
    n_workers: int,
    iteration: int = 0,
    key: int = 0,
) -> torch.Tensor:
    """Average one round's contributions for one key (engine.py:226-255).

    Quantized payloads are decoded, the vectors summed in ascending worker-id
    order in fp64 and divided by the worker count — one kernel launch. Mixing
    full and quantized contributions is a protocol violation."""
    if len(contributions) != n_workers:
        raise ProtocolViolation(
            f"iteration {iteration} key {key}: {len(contributions)} contributions, expected {n_workers}"
        )
    kinds = {kind for kind, _ in contributions.values()}
    if len(kinds) > 1:
        raise ProtocolViolation(f"iteration {iteration} key {key}: mixed full and quantized contributions")
    order = sorted(contributions)
    kind = kinds.pop()
    if kind == "quant":
        return dequantize_sum([contributions[w][1] for w in order])
    vecs = [_device_tensor(contributions[w][1]) for w in order]
    dtype = torch.float32 if all(v.dtype == torch.float32 for v in vecs) else torch.float64
    stacked = torch.stack([v.to(dtype) for v in vecs])
    n = stacked.shape[1]
    out = torch.empty(n, dtype=torch.float64, device=stacked.device)
    _lib.check(
        _lib.lib().cdsgd_aggregate_full(stacked.data_ptr(), _dt(stacked), len(vecs), n, n, out.data_ptr(), _stream()),
        "server_aggregate",
    )
    return out


def global_update(weights: KeyedVector, mean_grad: KeyedVector, eta_global: float) -> None:
    """Apply W <- W - eta * mean_grad in place (engine.py:258-265)."""
    if weights.layout != mean_grad.layout:
        raise LayoutError("mean gradient layout does not match the global weights")
    if eta_global < 0:
        raise ConfigError("eta_global must be ≥ 0")
    w, m = weights.values, mean_grad.values
    _lib.check(
        _lib.lib().cdsgd_global_update(w.data_ptr(), _dt(w), m.data_ptr(), _dt(m), w.shape[0], float(eta_global),
                                       _stream()),
        "global_update",
    )


def local_update(base_weights: KeyedVector, local_grad: KeyedVector, eta_local: float) -> KeyedVector:
    """Next local weights: last pulled global base minus one local gradient step (engine.py:268-274)."""
    if base_weights.layout != local_grad.layout:
        raise LayoutError("local gradient layout does not match the base weights")
    if eta_local < 0:
        raise ConfigError("eta_local must be ≥ 0")
    b, g = base_weights.values, local_grad.values
    out = torch.empty_like(b)
    _lib.check(
        _lib.lib().cdsgd_local_update(b.data_ptr(), _dt(b), g.data_ptr(), _dt(g), out.data_ptr(), _dt(out),
                                      b.shape[0], float(eta_local), _stream()),
        "local_update",
    )
    return KeyedVector(out, base_weights.layout)


__all__ = [
    "ALGORITHMS", "ConfigError", "ProtocolViolation", "SchedulingError", "HyperParams", "KeyedVector",
    "should_compress", "server_aggregate", "global_update", "local_update", "QuantizedPayload",
]
