"""Per-GPU CD-SGD worker: the fused quantize -> exchange -> apply step driver.

One process per GPU; each rank is one CD-SGD worker (Algorithm 1) AND a replica of
the parameter server: it keeps the global weights W (fp32, bitwise identical on
every rank), its own fp64 residual, local weights and packed-code buffers, and
drives the native ``cdsgd_engine`` of libcdsgd_b200.so (include/cdsgd_b200.h).

Semantics follow Worker/ServerNode/_run_lockstep (engine.py:288-663) with the
gradient supplied by the caller instead of ``loss_and_grad`` (engine.py:363):

    w = CDSGDWorker(layout, hp, w0, rank=r, comm=comm)
    for t in range(T):
        x = w.compute_weights()        # engine.py:335-343 (W during warm-up, else loc)
        g = my_gradient(x)             # fp32 CUDA tensor [layout.total]
        w.step(g)                      # K1 + exchange(t) || K2/K3(t-1) + local update
    w.flush()                          # W == W_T (ServerNode.weights after T rounds)

Round t's exchange runs on the engine's stream while the caller computes the
gradient of round t+1 at loc_{t+1} = W_t - eta_l * g_t (the paper's overlap).
Numeric errors are detected on the device and raised by ``check()`` (called by
``flush()`` and every ``check_every`` rounds) as CodecNumericError with the key,
key-local index and round; the residual is rolled back to the state before it.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from .codec import CodecNumericError, CorruptPayloadError, _locate
from .engine import ConfigError, HyperParams, SchedulingError
from .layout import Layout

_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


class _CudaBytes:
    """A raw device allocation seen as a uint8 CUDA array (torch.as_tensor aliases it)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


def _raw_stream(index: int) -> int:
    """cudaStream_t of the current torch stream on device `index` (the per-step host path:
    ~3 us cheaper than torch.cuda.current_stream(device).cuda_stream)."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(index)
    return torch.cuda.current_stream(index).cuda_stream


class CDSGDWorker:
    def __init__(
        self,
        layout: Layout,
        hp: HyperParams,
        init_weights,
        *,
        rank: int = 0,
        comm=None,
        force_compress: bool = False,
        bypass_local: bool = False,
        gnorm_ring: int = 64,
        check_every: int = 0,
        device=None,
        exchange: str = "p2p",
        group=None,
        weights: str = "f64",
        residual: str = "f64",
    ):
        if not torch.cuda.is_available():
            raise _lib.LibraryError("CDSGDWorker needs a CUDA device (no CPU fallback)")
        hp.validate()
        self.hp = hp
        self.layout = layout
        self.rank = rank
        self.world = hp.workers
        if self.world > 1 and comm is None:
            raise ConfigError("workers > 1 needs an NCCL Comm (paper_2106_10796_b200.comm.Comm)")
        if comm is not None and (comm.world != self.world or comm.rank != rank):
            raise ConfigError("comm size/rank do not match hp.workers/rank")
        self.comm = comm
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        dev = self.device
        n, nw = layout.total, layout.n_words
        w0 = init_weights if isinstance(init_weights, torch.Tensor) else torch.from_numpy(np.asarray(init_weights))
        if w0.numel() != n:
            raise ConfigError(f"initial weights have {w0.numel()} elements, layout needs {n}")
        if weights not in _lib.WEIGHTS:
            raise ConfigError(f"weights must be 'f64' (exact) or 'f32' (fast), got {weights!r}")
        self.weights_dtype = weights
        if residual not in _lib.RESIDUAL or (residual == "f32" and weights != "f32"):
            raise ConfigError("residual must be 'f64' (exact) or 'f32' (fast mode, with weights='f32')")
        self.residual_dtype = residual
        rt = torch.float64 if residual == "f64" else torch.float32
        wt = torch.float64 if weights == "f64" else torch.float32
        with torch.cuda.device(dev):
            self.W = w0.reshape(-1).to(device=dev, dtype=wt).clone()
            self.loc = w0.reshape(-1).to(device=dev, dtype=torch.float32).clone()
            self.residuals = [torch.zeros(n, dtype=rt, device=dev), torch.empty(n, dtype=rt, device=dev)]
            self.gathered = [torch.zeros(self.world * nw, dtype=torch.int32, device=dev).view(torch.uint32) for _ in range(2)]
            self.gsum = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(2)] if self.world > 1 else [None, None]
            self.err = torch.full((2,), -1, dtype=torch.int64, device=dev)
            self.gnorm_ring = max(int(gnorm_ring), 0)
            self.gnorm = torch.zeros(max(self.gnorm_ring, 1), dtype=torch.float64, device=dev)
            d = _lib.EngineDesc()
            d.algo = _lib.ALGO[hp.algo]
            d.nranks = self.world
            d.rank = rank
            d.k = hp.k
            d.warmup_n = hp.warmup_n
            d.force_compress = int(force_compress)
            d.bypass_local = int(bypass_local)
            d.gnorm_ring = self.gnorm_ring
            d.weights_dtype = _lib.WEIGHTS[weights]
            d.residual_dtype = _lib.RESIDUAL[residual]
            d.alpha = float(hp.alpha)
            d.eta_global = float(hp.eta_global)
            d.eta_local = float(hp.local_lr)
            d.weights = self.W.data_ptr()
            d.loc = self.loc.data_ptr()
            d.residual[0] = self.residuals[0].data_ptr()
            d.residual[1] = self.residuals[1].data_ptr()
            d.gathered[0] = self.gathered[0].data_ptr()
            d.gathered[1] = self.gathered[1].data_ptr()
            d.gsum[0] = self.gsum[0].data_ptr() if self.gsum[0] is not None else None
            d.gsum[1] = self.gsum[1].data_ptr() if self.gsum[1] is not None else None
            d.err = self.err.data_ptr()
            d.gnorm_sq = self.gnorm.data_ptr() if self.gnorm_ring else None
            self._desc = d
            out = C.c_void_p()
            _lib.check(
                _lib.lib().cdsgd_engine_create(C.byref(d), layout.handle(dev.index).ptr,
                                               comm.ptr if comm is not None else None, C.byref(out)),
                "cdsgd_engine_create",
            )
            self._eng = out
            self.exchange = exchange if self.world > 1 else "local"
            if self.world > 1 and exchange in ("p2p", "p2p-exact"):
                self._attach_p2p(group, exact=exchange == "p2p-exact")
            elif self.world > 1 and exchange != "nccl":
                raise ConfigError(f"exchange must be 'p2p', 'p2p-exact' or 'nccl', got {exchange!r}")
        self._keep: list = [None, None]  # the last two gradients: still read by in-flight rounds
        self._keep_ptr: list = [0, 0]
        self._nstep = 0
        self.check_every = int(check_every)
        self._since_check = 0
        self._lib = _lib.lib()

    def _attach_p2p(self, group, exact: bool = False) -> None:
        """Fused NVLink exchange: one symmetric buffer per rank, every peer's buffer mapped into
        this process; K1 stores codes straight into all ranks' slots and K2 synchronises on
        release/acquire flags (cdsgd_engine_attach_p2p). exact=True also replaces the
        correction all-reduce by the sharded fp64 NVLink reduce.

        The buffers are the library's own (cudaMalloc + CUDA IPC handles exchanged over the
        process group, cdsgd_p2p_buffer_*); CDSGD_P2P_MEMORY=torch uses torch's symmetric
        memory instead (a private torch API)."""
        import torch.distributed as dist

        lib = _lib.lib()
        n, nw = self.layout.total, self.layout.n_words
        nbytes = int(lib.cdsgd_p2p_bytes(self.world, n, nw))
        w_off = int(lib.cdsgd_p2p_weights_offset(self.world, n, nw))
        grp = group if group is not None else dist.group.WORLD
        self._p2p_group = grp
        if os.environ.get("CDSGD_P2P_MEMORY", "native") == "torch":
            import torch.distributed._symmetric_memory as symm_mem

            self._symm = symm_mem.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._symm.zero_()
            torch.cuda.synchronize(self.device)
            self._symm_handle = symm_mem.rendezvous(self._symm, grp)
            ptrs = [int(p) for p in self._symm_handle.buffer_ptrs]
        else:
            ptrs = self._native_symmetric(nbytes, grp)
        if len(ptrs) != self.world:
            raise ConfigError("symmetric memory group does not match hp.workers")
        arr = (C.c_void_p * self.world)(*ptrs)
        _lib.check(lib.cdsgd_engine_attach_p2p(self._eng, arr, self.world, int(exact)), "cdsgd_engine_attach_p2p")
        # with the exact correction the engine moved the W replica into the symmetric buffer (peers
        # write W' shards into it; CDSGD_W_SYMMETRIC=1: in every P2P mode, the engine's same rule),
        # and the code slots live there too (slot 0 at offset 0, slot 1 at the next 256-B boundary)
        if exact or os.environ.get("CDSGD_W_SYMMETRIC", "0") == "1":
            es = self.W.element_size()
            self.W = self._symm[w_off:w_off + es * n].view(self.W.dtype)
        slot = (self.world * nw * 4 + 255) // 256 * 256
        self.gathered = [self._symm[i * slot:i * slot + self.world * nw * 4].view(torch.uint32) for i in range(2)]
        torch.cuda.synchronize(self.device)
        dist.barrier(group=grp)  # every rank's flags are zero before any rank's first K1

    def _native_symmetric(self, nbytes: int, grp) -> list:
        """Allocate this rank's buffer, all-gather the IPC handles, map the peers' buffers.
        Returns the nranks base addresses (index = rank in the group)."""
        import torch.distributed as dist

        lib = _lib.lib()
        with torch.cuda.device(self.device):
            base = C.c_void_p()
            handle = (C.c_uint8 * _lib.P2P_HANDLE_BYTES)()
            _lib.check(lib.cdsgd_p2p_buffer_alloc(nbytes, C.byref(base), handle), "cdsgd_p2p_buffer_alloc")
            self._p2p_base = base.value
            handles = [None] * dist.get_world_size(grp)
            dist.all_gather_object(handles, bytes(handle), group=grp)
            me = dist.get_rank(grp)
            ptrs = []
            self._p2p_peers = []
            for r, h in enumerate(handles):
                if r == me:
                    ptrs.append(base.value)
                    continue
                hb = (C.c_uint8 * _lib.P2P_HANDLE_BYTES).from_buffer_copy(h)
                p = C.c_void_p()
                _lib.check(lib.cdsgd_p2p_buffer_open(hb, C.byref(p)), "cdsgd_p2p_buffer_open")
                self._p2p_peers.append(p.value)
                ptrs.append(p.value)
        self._symm = torch.as_tensor(_CudaBytes(base.value, nbytes), device=self.device)
        return ptrs

    def _release_symmetric(self) -> None:
        """Unmap the peers' buffers and free this rank's (after every rank stopped using it)."""
        base = getattr(self, "_p2p_base", None)
        if base is None:
            return
        import torch.distributed as dist

        torch.cuda.synchronize(self.device)
        if dist.is_available() and dist.is_initialized():
            dist.barrier(group=self._p2p_group)  # no rank's kernels still write into our buffer
        lib = _lib.lib()
        for p in self._p2p_peers:
            lib.cdsgd_p2p_buffer_close(C.c_void_p(p))
        self._p2p_peers = []
        self._symm = self.W = self.gathered = None
        lib.cdsgd_p2p_buffer_free(C.c_void_p(base))
        self._p2p_base = None

    # ------------------------------------------------------------------ state
    def state(self) -> _lib.EngineState:
        st = _lib.EngineState()
        _lib.check(self._lib.cdsgd_engine_get_state(self._eng, C.byref(st)), "engine_get_state")
        return st

    @property
    def t(self) -> int:
        return int(self.state().t)

    @property
    def residual(self) -> torch.Tensor:
        """The live residual (concatenated over keys): fp64, or fp32 in the fast mode."""
        return self.residuals[self.state().residual_index]

    @property
    def weights(self) -> torch.Tensor:
        """Global weights replica (W_t once every started round is applied, see flush()):
        fp64 in the exact mode (bitwise the reference's W on compressed rounds), fp32 in the
        fast mode."""
        return self.W

    def compute_weights(self) -> torch.Tensor:
        """Weights the next gradient must be computed at (engine.py:335-343)."""
        return self.loc if self.state().compute_is_loc else self.W

    @property
    def ce_fraction(self) -> float:
        """Share of each correction all-reduce carried by the copy engines (P2P mode)."""
        return float(self._lib.cdsgd_engine_ce_fraction(self._eng))

    def round_compressed(self, t: int) -> bool:
        r = self._lib.cdsgd_engine_round_compressed(self._eng, int(t))
        if r < 0:
            raise ConfigError(_lib.last_error())
        return bool(r)

    def round_payloads(self, t: int) -> list:
        """This rank's per-key QuantizedPayloads of compressed round t (engine.py:397-402),
        as views of the packed code buffer — valid until round t+2 reuses the slot. Feed them
        to ``wire.round_frames`` to talk to the reference ServerNode."""
        from .codec import QuantizedPayload

        if not (0 <= t < self.t) or t < self.t - 2:
            raise ConfigError(f"round {t} is not among the last two started rounds")
        if not self.round_compressed(t):
            raise ConfigError(f"round {t} pushed full-precision gradients, not codes")
        nw = self.layout.n_words
        mine = self.gathered[t % 2][self.rank * nw:(self.rank + 1) * nw]
        out, w0 = [], 0
        for span in self.layout.spans:
            k = (span.length + 15) // 16
            out.append(QuantizedPayload(mine[w0:w0 + k], self.hp.alpha, span.length))
            w0 += k
        return out

    def grad_norm(self, t: int) -> float:
        """||round-t mean gradient||_2 (engine.py:521); valid for the last gnorm_ring - 2 rounds."""
        if not self.gnorm_ring:
            raise ConfigError("grad-norm metric disabled (gnorm_ring=0)")
        return float(self.gnorm[t % self.gnorm_ring].sqrt().item())

    # ------------------------------------------------------------------ driving
    def step(self, grad: torch.Tensor) -> None:
        # Gradient buffers are usually reused (a training loop alternates two): a tensor that was
        # validated two rounds ago (the same object still held in _keep) skips the checks and
        # reuses its data pointer — on launch-bound layouts the per-call host cost is the limit.
        slot = self._nstep & 1
        if grad is self._keep[slot] and grad.data_ptr() == self._keep_ptr[slot]:
            ptr = self._keep_ptr[slot]
        else:
            if grad.dtype != torch.float32 or not grad.is_cuda or not grad.is_contiguous() or \
                    grad.numel() != self.layout.total:
                raise ConfigError("gradient must be a contiguous fp32 CUDA tensor of layout.total elements")
            ptr = grad.data_ptr()
        rc = self._lib.cdsgd_engine_step(self._eng, ptr, _raw_stream(self._dev_index))
        if rc != _lib.OK:
            msg = _lib.last_error()
            if rc == _lib.ERR_STATE:
                raise SchedulingError(msg)
            if rc == _lib.ERR_ARG:
                raise ConfigError(msg)
            raise _lib.LibraryError(msg, rc)
        self._keep[slot] = grad
        self._keep_ptr[slot] = ptr
        self._nstep += 1
        if self.check_every:
            self._since_check += 1
            if self._since_check >= self.check_every:
                self.check()

    def flush(self) -> None:
        """Apply the last exchanged round: afterwards W == W_t."""
        _lib.check(self._lib.cdsgd_engine_flush(self._eng, torch.cuda.current_stream(self.device).cuda_stream), "flush")
        self.check()

    def check(self) -> None:
        """Synchronise and raise the first device-side error (CodecNumericError / CorruptPayloadError)."""
        rnd, idx = C.c_int64(-1), C.c_int64(-1)
        rc = self._lib.cdsgd_engine_check(self._eng, torch.cuda.current_stream(self.device).cuda_stream,
                                          C.byref(rnd), C.byref(idx))
        self._since_check = 0
        if rc == _lib.OK:
            return
        if rc == _lib.ERR_NUMERIC:
            key, local = _locate(self.layout, int(idx.value))
            raise CodecNumericError(
                f"non-finite accumulated gradient at element {local} (key {key}, round {rnd.value})",
                local, key=key, round=int(rnd.value),
            )
        if rc == _lib.ERR_CORRUPT:
            raise CorruptPayloadError(_lib.last_error())
        if rc == _lib.ERR_PEER:
            raise _lib.PeerFailedError(_lib.last_error(), rc)
        raise _lib.LibraryError(_lib.last_error(), rc)

    def join(self, stream=None) -> None:
        """Make `stream` (default: current) wait for every exchange issued so far."""
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        _lib.check(self._lib.cdsgd_engine_join(self._eng, st), "join")

    def profile_begin(self) -> None:
        """Start recording CUDA events around every kernel / NCCL call of the step."""
        _lib.check(self._lib.cdsgd_engine_profile_begin(self._eng), "profile_begin")

    def profile_end(self) -> dict:
        """Per-kernel-class total ms and launch counts since profile_begin()."""
        out = (C.c_double * 22)()
        _lib.check(self._lib.cdsgd_engine_profile_end(self._eng, out), "profile_end")
        names = ("quantize", "apply_quant", "apply_full", "local_update", "exchange", "fused", "stage", "reduce",
                 "wait", "fused_local", "exchange_ce")
        return {nm: {"ms": out[2 * i], "n": int(out[2 * i + 1])} for i, nm in enumerate(names)}

    def close(self) -> None:
        """Destroy the engine; with the native symmetric buffer (P2P exchange) this is
        collective: every rank calls it (the buffer is freed after a barrier)."""
        if getattr(self, "_eng", None):
            _lib.lib().cdsgd_engine_destroy(self._eng)
            self._eng = None
        self._release_symmetric()

    def __del__(self):
        try:
            if getattr(self, "_eng", None):
                _lib.lib().cdsgd_engine_destroy(self._eng)
                self._eng = None
            # a native symmetric buffer is only released by an explicit (collective) close();
            # at interpreter exit the process's device memory goes with it
        except Exception:
            pass
