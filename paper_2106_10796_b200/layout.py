"""Key layouts: the contract that drives key-segmented packing.

Mirrors numcore.Layout / KeySpan / KeyedVector (reference numcore.py:40-115):
a flat parameter vector partitioned into contiguous per-tensor keys, key ids
dense 0..K-1, every key of length >= 1. Packing restarts at each key because the
reference quantizes key by key (engine.py:397-402), so the packed buffer of a
layout is the concatenation of ceil(len_k/16) words per key.

Also provides the gradient layouts the benchmarks are quoted on:
ResNet-20/CIFAR (59 keys, 269,722), ResNet-50 (161 keys, 25,557,032) and
VGG-16 (32 keys, 138,357,544), in torchvision parameter order.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

from . import _lib


class LayoutError(ValueError):
    """Mismatched key layouts or a malformed key table (numcore.py:28-29)."""


@dataclass(frozen=True)
class KeySpan:
    key: int
    name: str
    start: int
    length: int


class Layout:
    """Contiguous, non-overlapping partition of a flat vector into keys (numcore.py:48-84)."""

    def __init__(self, sizes: Sequence[tuple[str, int]]):
        spans = []
        offset = 0
        for key, (name, length) in enumerate(sizes):
            length = int(length)
            if length < 1:
                raise LayoutError(f"key {name!r} has non-positive length {length}")
            spans.append(KeySpan(key, name, offset, length))
            offset += length
        if not spans:
            raise LayoutError("layout needs at least one key")
        self.spans: tuple[KeySpan, ...] = tuple(spans)
        self.total: int = offset
        self.n_words: int = sum((s.length + 15) // 16 for s in spans)
        self._handles: dict[int, "_DeviceLayout"] = {}

    @classmethod
    def from_lengths(cls, lengths: Sequence[int], prefix: str = "k") -> "Layout":
        return cls([(f"{prefix}{i}", int(n)) for i, n in enumerate(lengths)])

    @property
    def lengths(self) -> list[int]:
        return [s.length for s in self.spans]

    def slice(self, key: int) -> slice:
        span = self.spans[key]
        return slice(span.start, span.start + span.length)

    def word_slice(self, key: int) -> slice:
        start = sum((s.length + 15) // 16 for s in self.spans[:key])
        return slice(start, start + (self.spans[key].length + 15) // 16)

    @property
    def keys(self) -> range:
        return range(len(self.spans))

    def __len__(self) -> int:
        return len(self.spans)

    def __eq__(self, other) -> bool:
        return isinstance(other, Layout) and self.spans == other.spans

    def __hash__(self) -> int:
        return hash(self.spans)

    def __repr__(self) -> str:
        inner = ", ".join(f"{s.name}[{s.length}]" for s in self.spans)
        return f"Layout({inner})"

    def handle(self, device: int | None = None) -> "_DeviceLayout":
        """Device-resident key table for the current (or given) CUDA device."""
        import torch

        dev = torch.cuda.current_device() if device is None else int(device)
        h = self._handles.get(dev)
        if h is None:
            with torch.cuda.device(dev):
                h = _DeviceLayout(self.lengths)
            self._handles[dev] = h
        return h


class _DeviceLayout:
    """Owner of a ``cdsgd_layout*`` (cdsgd_layout_create/destroy)."""

    def __init__(self, lengths: Sequence[int]):
        lib = _lib.lib()
        arr = (C.c_int64 * len(lengths))(*[int(x) for x in lengths])
        out = C.c_void_p()
        _lib.check(lib.cdsgd_layout_create(arr, len(lengths), C.byref(out)), "cdsgd_layout_create")
        self.ptr = out
        self.n = int(lib.cdsgd_layout_elems(out))
        self.n_words = int(lib.cdsgd_layout_words(out))

    def __del__(self):
        try:
            if self.ptr:
                _lib.lib().cdsgd_layout_destroy(self.ptr)
        except Exception:
            pass


def single(n: int, name: str = "w") -> Layout:
    return Layout([(name, n)])


def resnet20_cifar() -> Layout:
    """ResNet-20 for CIFAR-10 (He et al. 2016, option-A shortcuts): 59 keys, 269,722."""
    sizes: list[tuple[str, int]] = [("conv1.weight", 16 * 3 * 9), ("bn1.weight", 16), ("bn1.bias", 16)]
    cin = 16
    for stage, cout in enumerate((16, 32, 64), start=1):
        for b in range(3):
            c_in = cin if b == 0 else cout
            p = f"layer{stage}.{b}."
            sizes += [
                (p + "conv1.weight", cout * c_in * 9), (p + "bn1.weight", cout), (p + "bn1.bias", cout),
                (p + "conv2.weight", cout * cout * 9), (p + "bn2.weight", cout), (p + "bn2.bias", cout),
            ]
        cin = cout
    sizes += [("fc.weight", 64 * 10), ("fc.bias", 10)]
    return Layout(sizes)


def resnet50() -> Layout:
    """torchvision ResNet-50 parameters in registration order: 161 keys, 25,557,032."""
    sizes: list[tuple[str, int]] = [("conv1.weight", 64 * 3 * 49), ("bn1.weight", 64), ("bn1.bias", 64)]
    inplanes = 64
    for stage, (planes, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3)), start=1):
        for b in range(blocks):
            p = f"layer{stage}.{b}."
            width, out = planes, planes * 4
            sizes += [
                (p + "conv1.weight", width * inplanes), (p + "bn1.weight", width), (p + "bn1.bias", width),
                (p + "conv2.weight", width * width * 9), (p + "bn2.weight", width), (p + "bn2.bias", width),
                (p + "conv3.weight", out * width), (p + "bn3.weight", out), (p + "bn3.bias", out),
            ]
            if b == 0:
                sizes += [(p + "downsample.0.weight", out * inplanes), (p + "downsample.1.weight", out),
                          (p + "downsample.1.bias", out)]
            inplanes = out
    sizes += [("fc.weight", 1000 * 2048), ("fc.bias", 1000)]
    return Layout(sizes)


def vgg16() -> Layout:
    """torchvision VGG-16 (no BN) parameters: 32 keys, 138,357,544."""
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    sizes: list[tuple[str, int]] = []
    cin, idx = 3, 0
    for v in cfg:
        if v == "M":
            idx += 1
            continue
        sizes += [(f"features.{idx}.weight", v * cin * 9), (f"features.{idx}.bias", v)]
        cin = v
        idx += 2
    for i, (fi, fo) in zip((0, 3, 6), ((512 * 7 * 7, 4096), (4096, 4096), (4096, 1000))):
        sizes += [(f"classifier.{i}.weight", fo * fi), (f"classifier.{i}.bias", fo)]
    return Layout(sizes)


def from_module(module) -> Layout:
    """Per-parameter key table of a torch.nn.Module (one key per parameter tensor)."""
    sizes = [(name, p.numel()) for name, p in module.named_parameters() if p.requires_grad]
    return Layout(sizes)


NAMED = {"resnet20": resnet20_cifar, "resnet50": resnet50, "vgg16": vgg16}


def by_name(name: str) -> Layout:
    if name in NAMED:
        return NAMED[name]()
    if name.startswith("single:"):
        return single(int(float(name.split(":", 1)[1])))
    if name.startswith("keys:"):
        return Layout.from_lengths([int(x) for x in name.split(":", 1)[1].split(",")])
    raise LayoutError(f"unknown layout {name!r}")
