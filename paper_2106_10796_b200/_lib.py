"""ctypes binding of libcdsgd_b200.so (the C ABI in include/cdsgd_b200.h).

This is the same binding a maintainer would add to the reference package (see
INTEGRATION.md). There is no fallback: if the library is missing or CUDA is
unavailable, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CDSGD_LIB: load another build of the same library (development A/B of kernel variants)
LIB_PATH = os.environ.get("CDSGD_LIB") or os.path.join(_HERE, "libcdsgd_b200.so")

OK = 0
ERR_ARG, ERR_CUDA, ERR_NCCL, ERR_STATE, ERR_NUMERIC, ERR_CORRUPT, ERR_PEER = -1, -2, -3, -4, -5, -6, -7
NO_ERROR = 0xFFFFFFFFFFFFFFFF
INDEX_BITS = 40
F32, F64 = 0, 1
ALGO = {"ssgd": 0, "lusgd": 1, "bitsgd": 2, "cdsgd": 3}
UNIQUE_ID_BYTES = 128
ABI_VERSION = 2
WEIGHTS = {"f64": 1, "f32": 0}  # CDSGD_F64 (exact, default) / CDSGD_F32 (fast)
RESIDUAL = WEIGHTS  # residual_dtype: f64 exact (default) / f32 fast mode (needs fp32 weights)

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
u64 = C.c_uint64
f64 = C.c_double


class EngineDesc(C.Structure):
    _fields_ = [
        ("algo", i32), ("nranks", i32), ("rank", i32), ("k", i32), ("warmup_n", i32),
        ("force_compress", i32), ("bypass_local", i32), ("gnorm_ring", i32), ("weights_dtype", i32),
        ("residual_dtype", i32),
        ("alpha", f64), ("eta_global", f64), ("eta_local", f64),
        ("weights", vp), ("loc", vp), ("residual", vp * 2), ("gathered", vp * 2), ("gsum", vp * 2),
        ("err", vp), ("gnorm_sq", vp),
    ]


class EngineState(C.Structure):
    _fields_ = [
        ("t", i64), ("residual_index", i32), ("compute_is_loc", i32), ("pending", i32),
        ("last_compressed", i32), ("failed", i32),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "cdsgd_abi_version": (C.c_int, []),
    "cdsgd_last_error": (C.c_char_p, []),
    "cdsgd_launch_count": (u64, []),
    "cdsgd_layout_create": (C.c_int, [C.POINTER(i64), i32, C.POINTER(vp)]),
    "cdsgd_layout_destroy": (C.c_int, [vp]),
    "cdsgd_layout_elems": (i64, [vp]),
    "cdsgd_layout_words": (i64, [vp]),
    "cdsgd_layout_keys": (i32, [vp]),
    "cdsgd_layout_offsets": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64)]),
    "cdsgd_quantize": (C.c_int, [vp, vp, i32, vp, vp, vp, f64, vp, u64, vp]),
    "cdsgd_dequantize_sum": (C.c_int, [vp, vp, i32, i64, f64, vp, vp, vp]),
    "cdsgd_aggregate_full": (C.c_int, [vp, i32, i32, i64, i64, vp, vp]),
    "cdsgd_pack_symbols": (C.c_int, [vp, i64, vp, vp, vp]),
    "cdsgd_unpack_symbols": (C.c_int, [vp, i64, vp, vp]),
    "cdsgd_global_update": (C.c_int, [vp, i32, vp, i32, i64, f64, vp]),
    "cdsgd_local_update": (C.c_int, [vp, i32, vp, i32, vp, i32, i64, f64, vp]),
    "cdsgd_apply_quant": (C.c_int, [vp, vp, i32, vp, i32, i64, f64, f64, vp, vp, f64, vp, u64, vp, vp]),
    "cdsgd_apply_full": (C.c_int, [vp, i32, vp, i32, i64, f64, vp, vp, f64, vp, u64, vp, vp]),
    "cdsgd_fused_round": (C.c_int, [vp, vp, vp, vp, i32, vp, f64, vp, u64, vp, i32, vp, vp, i32, i64, f64, f64, u64, vp,
                                    vp]),
    "cdsgd_quantize_f32r": (C.c_int, [vp, vp, vp, vp, vp, f64, vp, u64, vp]),
    "cdsgd_comm_unique_id": (C.c_int, [vp]),
    "cdsgd_comm_init": (C.c_int, [vp, i32, i32, C.POINTER(vp)]),
    "cdsgd_comm_destroy": (C.c_int, [vp]),
    "cdsgd_allgather_words": (C.c_int, [vp, vp, vp, i64, vp]),
    "cdsgd_allreduce_sum_f32": (C.c_int, [vp, vp, vp, i64, vp]),
    "cdsgd_engine_create": (C.c_int, [C.POINTER(EngineDesc), vp, vp, C.POINTER(vp)]),
    "cdsgd_engine_destroy": (C.c_int, [vp]),
    "cdsgd_engine_step": (C.c_int, [vp, vp, vp]),
    "cdsgd_engine_flush": (C.c_int, [vp, vp]),
    "cdsgd_engine_get_state": (C.c_int, [vp, C.POINTER(EngineState)]),
    "cdsgd_engine_check": (C.c_int, [vp, vp, C.POINTER(i64), C.POINTER(i64)]),
    "cdsgd_engine_round_compressed": (C.c_int, [vp, i64]),
    "cdsgd_engine_join": (C.c_int, [vp, vp]),
    "cdsgd_p2p_bytes": (i64, [i32, i64, i64]),
    "cdsgd_p2p_weights_offset": (i64, [i32, i64, i64]),
    "cdsgd_engine_attach_p2p": (C.c_int, [vp, C.POINTER(vp), i32, i32]),
    "cdsgd_p2p_buffer_alloc": (C.c_int, [i64, C.POINTER(vp), vp]),
    "cdsgd_p2p_buffer_open": (C.c_int, [vp, C.POINTER(vp)]),
    "cdsgd_p2p_buffer_close": (C.c_int, [vp]),
    "cdsgd_p2p_buffer_free": (C.c_int, [vp]),
    "cdsgd_engine_profile_begin": (C.c_int, [vp]),
    "cdsgd_engine_profile_end": (C.c_int, [vp, C.POINTER(f64)]),
    "cdsgd_engine_ce_fraction": (C.c_double, [vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)
P2P_HANDLE_BYTES = 64  # CDSGD_P2P_HANDLE_BYTES (a cudaIpcMemHandle_t)

_lib = None


class LibraryError(RuntimeError):
    """The CUDA extension is missing or returned an error."""

    def __init__(self, message: str, code: int = ERR_CUDA):
        super().__init__(message)
        self.code = code


class PeerFailedError(LibraryError):
    """Another rank of the exchange failed (its flags arrived poisoned); this rank applied
    nothing after that round. The failing rank raises the cause (e.g. CodecNumericError)."""


def load(path: str = LIB_PATH):
    """Load the shared library (no GPU needed just to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cdsgd_abi_version() != ABI_VERSION:
        raise LibraryError("libcdsgd_b200.so ABI version mismatch")
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load()


def last_error() -> str:
    return lib().cdsgd_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status != OK:
        raise LibraryError(f"{what}: {last_error()}" if what else last_error(), status)


def launch_count() -> int:
    return int(lib().cdsgd_launch_count())
