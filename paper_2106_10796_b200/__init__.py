"""B200-native CD-SGD hot path (arXiv 2106.10796): 2-bit error-feedback quantizer,
NCCL exchange of packed codes, fused delayed update with k-step correction.

Public modules mirror the reference package ``cdsgd``:
  codec   — quantize / dequantize / pack_symbols / unpack_symbols / payload accounting
  engine  — HyperParams / should_compress / server_aggregate / global_update / local_update
  layout  — Layout / KeySpan (+ ResNet-20/50, VGG-16 gradient layouts)
  worker  — CDSGDWorker, the per-GPU fused step driver (native engine)
  comm    — NCCL communicator bootstrap
All compute runs in libcdsgd_b200.so (sm_100a); there is no CPU fallback.
"""

from . import _lib  # noqa: F401

__version__ = "0.1.0"


def load_library():
    """Load libcdsgd_b200.so; raises if it has not been built."""
    return _lib.load()
