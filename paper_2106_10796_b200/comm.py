"""NCCL communicator owned by libcdsgd_b200.so, bootstrapped over torch.distributed.

Replaces the reference's parameter-server transports (in-process queues and TCP,
protocol.py:174-288; engine.py:614-766): one process per GPU, the packed codes
are all-gathered and correction gradients all-reduced by NCCL over NVLink /
NVSwitch. torch.distributed (any backend, e.g. gloo or nccl) only carries the
128-byte ncclUniqueId from rank 0 to the others — plumbing, not data path.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib


def unique_id() -> bytes:
    buf = C.create_string_buffer(_lib.UNIQUE_ID_BYTES)
    _lib.check(_lib.lib().cdsgd_comm_unique_id(buf), "ncclGetUniqueId")
    return buf.raw


def share_unique_id(rank: int, make=unique_id, group=None) -> bytes:
    """Rank 0 creates the id; every rank returns the same 128 bytes."""
    import torch.distributed as dist

    obj = [make() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != _lib.UNIQUE_ID_BYTES:
        raise _lib.LibraryError("bad NCCL unique id received")
    return bytes(uid)


class Comm:
    """A ``cdsgd_comm*`` (ncclComm_t) for this rank on the current CUDA device."""

    def __init__(self, uid: bytes, world: int, rank: int):
        if not torch.cuda.is_available():
            raise _lib.LibraryError("NCCL exchange needs a CUDA device")
        out = C.c_void_p()
        _lib.check(_lib.lib().cdsgd_comm_init(uid, world, rank, C.byref(out)), "ncclCommInitRank")
        self.ptr = out
        self.world = world
        self.rank = rank

    @classmethod
    def from_torch_distributed(cls, group=None) -> "Comm":
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        return cls(share_unique_id(rank, group=group), world, rank)

    def allgather_words(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        _lib.check(
            _lib.lib().cdsgd_allgather_words(self.ptr, send.data_ptr(), recv.data_ptr(), send.numel(),
                                             torch.cuda.current_stream().cuda_stream),
            "allgather",
        )

    def allreduce_sum(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        _lib.check(
            _lib.lib().cdsgd_allreduce_sum_f32(self.ptr, send.data_ptr(), recv.data_ptr(), send.numel(),
                                               torch.cuda.current_stream().cuda_stream),
            "allreduce",
        )

    def close(self) -> None:
        if getattr(self, "ptr", None):
            _lib.lib().cdsgd_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
