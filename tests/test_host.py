"""CPU-only checks of the host layer: the C-ABI library loads and exports every
symbol include/cdsgd_b200.h declares, layouts match the named models, and the
reference-mirroring host logic (HyperParams, should_compress, payload accounting)
behaves like the reference. No compute call is made without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "cdsgd_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\*?\s+\**(cdsgd_[a-z0-9_]+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2106_10796_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED_SYMBOLS)
    assert lib.cdsgd_abi_version() == _lib.ABI_VERSION == 2


def test_library_is_sm100a():
    import subprocess

    from paper_2106_10796_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "LDG.E.NA.ENL2.256" in sass  # 256-bit residual loads in K1


def test_layout_create_without_gpu_fails_cleanly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2106_10796_b200 import _lib

    lib = _lib.load()
    out = ctypes.c_void_p()
    arr = (ctypes.c_int64 * 2)(5, 0)
    assert lib.cdsgd_layout_create(arr, 2, ctypes.byref(out)) == _lib.ERR_ARG
    assert "non-positive" in _lib.last_error()


def test_named_layouts():
    from paper_2106_10796_b200 import layout as L

    r20, r50, vgg = L.resnet20_cifar(), L.resnet50(), L.vgg16()
    assert (len(r20), r20.total, r20.n_words) == (59, 269722, 16858)
    assert (len(r50), r50.total, r50.n_words) == (161, 25557032, 1597315)
    assert (len(vgg), vgg.total, vgg.n_words) == (32, 138357544, 8647347)
    assert [s for s in r50.lengths if s % 16] == [1000]


def test_named_layouts_match_torchvision():
    tv = pytest.importorskip("torchvision")
    from paper_2106_10796_b200 import layout as L

    for got, m in ((L.resnet50(), tv.models.resnet50()), (L.vgg16(), tv.models.vgg16())):
        ref = L.from_module(m)
        assert [(s.name, s.length) for s in got.spans] == [(s.name, s.length) for s in ref.spans]


def test_layout_semantics():
    from paper_2106_10796_b200.layout import Layout, LayoutError

    lay = Layout([("a", 17), ("b", 1), ("c", 32)])
    assert lay.total == 50 and lay.n_words == 2 + 1 + 2
    assert lay.slice(1) == slice(17, 18) and lay.word_slice(2) == slice(3, 5)
    with pytest.raises(LayoutError):
        Layout([("a", 0)])
    with pytest.raises(LayoutError):
        Layout([])


def test_hyperparams_and_schedule():
    from paper_2106_10796_b200 import engine as E

    with pytest.raises(E.ConfigError):
        E.HyperParams(algo="adam").validate()
    with pytest.raises(E.ConfigError):
        E.HyperParams(algo="cdsgd", k=0).validate()
    hp = E.HyperParams(algo="cdsgd", eta_global=0.1).validate()
    assert hp.local_lr == 0.1 and hp.k == 5 and hp.alpha == 0.5 and hp.warmup_n == 5
    assert [E.should_compress(c, 4) for c in (1, 2, 3, 4)] == [True, True, True, False]
    assert sum(E.should_compress(c, 5) for c in range(1, 21)) == 16
    with pytest.raises(E.ConfigError):
        E.should_compress(0, 4)


def test_payload_accounting():
    from paper_2106_10796_b200 import codec as cx

    assert cx.payload_bytes(0) == 0 and cx.payload_bytes(16) == 4 and cx.payload_bytes(17) == 8
    assert cx.compression_ratio(16) == 16.0 and cx.compression_ratio(17) == 8.5 and cx.compression_ratio(0) == 1.0
    assert cx.serialized_payload_bytes(16384) == 4109
    with pytest.raises(cx.CodecError):
        cx.payload_bytes(-1)


def test_payload_serialization_roundtrip_host(codec_golden):
    from paper_2106_10796_b200 import codec as cx

    G = codec_golden
    for name in G["q_names"]:
        blob = G[f"q_{name}_bytes"].tobytes()
        p = cx.QuantizedPayload.from_bytes(blob, device="cpu")
        assert p.to_bytes() == blob
        assert np.array_equal(p.words.numpy(), G[f"q_{name}_words"])
    with pytest.raises(cx.CorruptPayloadError):
        cx.QuantizedPayload.from_bytes(b"\x03" + blob[1:], device="cpu")
    with pytest.raises(cx.CorruptPayloadError):
        cx.QuantizedPayload.from_bytes(blob[:-1], device="cpu")
    with pytest.raises(cx.CorruptPayloadError):
        cx.QuantizedPayload(np.zeros(2, np.uint32), 0.5, 40)


def test_compute_paths_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2106_10796_b200 import _lib, codec as cx

    with pytest.raises(_lib.LibraryError):
        cx.ResidualState.zeros(8)
    with pytest.raises(_lib.LibraryError):
        cx.quantize(cx.ResidualState.__new__(cx.ResidualState), np.zeros(4, np.float32), 0.5)
