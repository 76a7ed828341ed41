"""Real-model integration: train a torch.nn.Module with CD-SGD.

The reference computes gradients with its own toy models (``loss_and_grad``,
numcore.py:272-318) and keeps one key per parameter tensor (numcore.py:199-211). Here any
module's parameters become the key layout (registration order, one key per tensor),
autograd accumulates straight into the worker's flat fp32 gradient buffer (each
``param.grad`` is a view of it — no gather copy), and after every round the weights
the next gradient must be computed at (W during warm-up, the local weights after,
engine.py:335-343) are loaded back into the parameters.

    m = CDSGDModule(model, HyperParams(algo="cdsgd", eta_global=0.1, eta_local=0.4, k=4))
    for x, y in data:
        loss_fn(m.module(x), y).backward()   # grads land in the worker's buffer
        m.step()                              # quantize + exchange + delayed update
    m.flush()                                 # model parameters <- global weights W_T
"""

from __future__ import annotations

import torch

from .engine import HyperParams
from .layout import from_module
from .worker import CDSGDWorker


class CDSGDModule:
    def __init__(self, module: torch.nn.Module, hp: HyperParams, *, rank: int = 0, comm=None,
                 exchange: str = "p2p", device=None, **worker_kw):
        self.module = module
        self.params = [p for p in module.parameters() if p.requires_grad]
        if any(p.dtype != torch.float32 for p in self.params):
            raise TypeError("CD-SGD weights are fp32 (the codec itself runs in fp64)")
        self.layout = from_module(module)
        self._view_cache = {}
        dev = torch.device(device) if device is not None else self.params[0].device
        w0 = torch.empty(self.layout.total, dtype=torch.float32, device=dev)
        with torch.no_grad():
            for v, p in zip(self._make_views(w0), self.params):
                v.copy_(p.detach())
        self.worker = CDSGDWorker(self.layout, hp, w0, rank=rank, comm=comm, exchange=exchange, device=dev,
                                  **worker_kw)
        # round t's gradient stays readable until round t+1 is applied: two buffers alternate
        self._grads = [torch.zeros(self.layout.total, dtype=torch.float32, device=dev) for _ in range(2)]
        self._bind_grads(0)
        self._load(self.worker.compute_weights())

    def _views(self, flat: torch.Tensor):
        """Cached per buffer: the SAME view objects are bound as .grad, so step() can tell
        by identity that autograd accumulated in place (no copy)."""
        key = (flat.data_ptr(), flat.numel())
        v = self._view_cache.get(key)
        if v is None:
            v = self._view_cache[key] = self._make_views(flat)
        return v

    def _make_views(self, flat: torch.Tensor):
        """Each parameter's key as a view of a flat buffer with the PARAMETER's strides, so a
        channels_last weight keeps its memory order in W / loc / the gradient (the codec is
        elementwise per key: element order inside a key is the caller's choice). Parameter
        loads and autograd's gradient accumulation then need no layout conversion."""
        out = []
        for s, p in zip(self.layout.spans, self.params):
            if p.is_contiguous() or not (p.dim() == 4 and p.is_contiguous(memory_format=torch.channels_last)):
                out.append(flat[s.start:s.start + s.length].view_as(p))
            else:
                out.append(flat.as_strided(p.shape, p.stride(), flat.storage_offset() + s.start))
        return out

    def _bind_grads(self, i: int) -> None:
        buf = self._grads[i]
        buf.zero_()
        for p, v in zip(self.params, self._views(buf)):
            p.grad = v

    def _load(self, flat: torch.Tensor) -> None:
        # one multi-tensor launch instead of a copy per parameter (ResNet-50: 161 launches);
        # fp64 global weights (exact mode: warm-up rounds, flush) are rounded to fp32 first
        if flat.dtype != torch.float32:
            views = self._make_views(flat.to(torch.float32))  # a temporary: not cached
        else:
            views = self._views(flat)
        with torch.no_grad():
            torch._foreach_copy_(self.params, views)

    @property
    def t(self) -> int:
        return self.worker.t

    def step(self) -> None:
        """Push this round's gradient (the module's .grad) and move to the next round."""
        t = self.worker.t
        g = self._grads[t % 2]
        for p, v in zip(self.params, self._views(g)):
            if p.grad is not v and p.grad is not None:
                with torch.no_grad():
                    v.copy_(p.grad)  # an optimizer or user replaced .grad: fall back to a copy
        self.worker.step(g)
        self._bind_grads((t + 1) % 2)
        self._load(self.worker.compute_weights())

    def flush(self) -> None:
        """Apply the last round and load the global weights W into the module."""
        self.worker.flush()
        self._load(self.worker.weights)

    def grad_norm(self, t: int) -> float:
        return self.worker.grad_norm(t)
