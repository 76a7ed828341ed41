"""Real-model integration: train a torch.nn.Module with CD-SGD.

The reference computes gradients with its own toy models (``loss_and_grad``,
numcore.py:272-318) and keeps one key per parameter tensor (numcore.py:199-211). Here any
module's parameters become the key layout (registration order, one key per tensor),
autograd accumulates straight into the worker's flat fp32 gradient buffer (each
``param.grad`` is a view of it — no gather copy), and after every round the weights the
next gradient must be computed at (W during warm-up, the local weights after,
engine.py:335-343) are loaded back into the parameters.

    m = CDSGDModule(model, HyperParams(algo="cdsgd", eta_global=0.1, eta_local=0.4, k=4), buckets=4)
    for x, y in data:
        loss_fn(m.module(x), y).backward()   # grads land in the workers' buffers; with buckets
                                              # the exchange starts during backward
        m.step()                              # finish the round
    m.flush()                                 # model parameters <- global weights W_T

Layer-wise pipelining (the paper quantizes and exchanges layer by layer as
backward produces each gradient). With ``buckets=B > 1`` the parameters are grouped, in
reverse registration order (backward produces the last layers first), into B buckets of
about equal size, each driven by its own CDSGDWorker on a side stream. A
post-accumulate-grad hook counts each bucket's parameters in; when the last one has its
gradient, the bucket's step (quantize + exchange + delayed apply + local update + reload of
its compute weights) is issued on the side stream behind an event, so it runs while
backward continues with the earlier layers on the main stream. ``step()`` then makes the
main stream wait for every bucket. The semantics are exactly the unbucketed ones: the
reference quantizes, aggregates and commits every key independently (engine.py:397-402,
509-514), and every bucket follows the same round schedule; only the per-round grad norm
(engine.py:521) is summed over buckets. One backward per step when pipelined.

Element order inside a key: ``memory_order="reference"`` (default) flattens every
parameter in its logical (contiguous) order — the reference's — so round payloads and wire
frames (``wire.round_frames``) match what a reference worker would push for the same
gradient. ``memory_order="param"`` instead views each key with the parameter's own strides
(channels_last weights keep their memory order: no layout conversion on load / gradient
accumulation; the codec is elementwise, so the round math is unchanged, but a key's element
order then differs from the reference's flatten order).
"""

from __future__ import annotations

import torch

from .engine import ConfigError, HyperParams
from .layout import Layout
from .worker import CDSGDWorker


class _Bucket:
    """A group of parameters with one CDSGDWorker over their keys."""

    def __init__(self, params, names, hp, dev, order, worker_kw, rank, comm, exchange):
        self.params = params
        self.layout = Layout([(nm, p.numel()) for nm, p in zip(names, params)])
        self.order = order
        self._cache = {}
        w0 = torch.empty(self.layout.total, dtype=torch.float32, device=dev)
        with torch.no_grad():
            for v, p in zip(self.make_views(w0), params):
                v.copy_(p.detach())
        self.worker = CDSGDWorker(self.layout, hp, w0, rank=rank, comm=comm, exchange=exchange, device=dev,
                                  **worker_kw)
        # round t's gradient stays readable until round t+1 is applied: two buffers alternate
        self.grads = [torch.zeros(self.layout.total, dtype=torch.float32, device=dev) for _ in range(2)]
        self.pending = len(params)
        self.fired = False
        self.done = torch.cuda.Event()

    def make_views(self, flat):
        out = []
        for s, p in zip(self.layout.spans, self.params):
            cl = self.order == "param" and p.dim() == 4 and not p.is_contiguous() and \
                p.is_contiguous(memory_format=torch.channels_last)
            if cl:
                out.append(flat.as_strided(p.shape, p.stride(), flat.storage_offset() + s.start))
            else:
                out.append(flat[s.start:s.start + s.length].view(p.shape))
        return out

    def views(self, flat):
        """Cached per buffer: the SAME view objects are bound as .grad, so step() can tell by
        identity that autograd accumulated in place (no copy)."""
        key = (flat.data_ptr(), flat.numel())
        v = self._cache.get(key)
        if v is None:
            v = self._cache[key] = self.make_views(flat)
        return v

    def bind_grads(self, i: int) -> None:
        buf = self.grads[i]
        buf.zero_()
        for p, v in zip(self.params, self.views(buf)):
            p.grad = v

    def load(self, flat) -> None:
        # one multi-tensor launch per bucket; fp64 global weights (exact mode: warm-up rounds,
        # flush) are rounded to fp32 first
        views = self.make_views(flat.to(torch.float32)) if flat.dtype != torch.float32 else self.views(flat)
        with torch.no_grad():
            torch._foreach_copy_(self.params, views)

    def step(self) -> None:
        t = self.worker.t
        g = self.grads[t % 2]
        for p, v in zip(self.params, self.views(g)):
            if p.grad is not v and p.grad is not None:
                with torch.no_grad():
                    v.copy_(p.grad)  # an optimizer or user replaced .grad: fall back to a copy
        self.worker.step(g)
        self.bind_grads((t + 1) % 2)
        self.load(self.worker.compute_weights())


class CDSGDModule:
    def __init__(self, module: torch.nn.Module, hp: HyperParams, *, rank: int = 0, comm=None,
                 exchange: str = "p2p", device=None, buckets: int = 1, pipelined: bool | None = None,
                 memory_order: str = "reference", **worker_kw):
        self.module = module
        named = [(n, p) for n, p in module.named_parameters() if p.requires_grad]
        self.names = [n for n, _ in named]
        self.params = [p for _, p in named]
        if any(p.dtype != torch.float32 for p in self.params):
            raise TypeError("CD-SGD weights are fp32 (the codec itself runs in fp64)")
        if memory_order not in ("reference", "param"):
            raise ConfigError("memory_order must be 'reference' or 'param'")
        if buckets < 1:
            raise ConfigError("buckets must be >= 1")
        self.layout = Layout([(n, p.numel()) for n, p in named])  # every key, registration order
        dev = torch.device(device) if device is not None else self.params[0].device
        self.device = dev
        self.pipelined = (buckets > 1) if pipelined is None else bool(pipelined)
        # buckets in reverse registration order (backward's order), ~equal element counts
        groups, cur, tot = [], [], 0
        target = self.layout.total / buckets
        for i in reversed(range(len(self.params))):
            cur.append(i)
            tot += self.params[i].numel()
            if tot >= target * (len(groups) + 1) and len(groups) < buckets - 1:
                groups.append(cur)
                cur = []
        if cur:
            groups.append(cur)
        self.buckets = []
        self._bucket_of = {}
        for grp in groups:
            idx = sorted(grp)
            b = _Bucket([self.params[i] for i in idx], [self.names[i] for i in idx], hp, dev, memory_order, worker_kw,
                        rank, comm, exchange)
            self.buckets.append(b)
            for i in idx:
                self._bucket_of[id(self.params[i])] = b
        self._side = torch.cuda.Stream(dev) if self.pipelined else None
        self._hooks = []
        if self.pipelined:
            for p in self.params:
                self._hooks.append(p.register_post_accumulate_grad_hook(self._on_grad))
        for b in self.buckets:
            b.bind_grads(0)
            b.load(b.worker.compute_weights())

    # ------------------------------------------------------------------ compatibility
    @property
    def worker(self) -> CDSGDWorker:
        """The worker of a single-bucket module (engine state, grad norms, round payloads)."""
        if len(self.buckets) != 1:
            raise ConfigError("a bucketed module has one worker per bucket: see .buckets")
        return self.buckets[0].worker

    @property
    def t(self) -> int:
        return self.buckets[0].worker.t

    # ------------------------------------------------------------------ pipelined rounds
    def _fire(self, b: _Bucket) -> None:
        """Issue bucket b's round on the side stream behind everything enqueued so far on the
        current (backward) stream — its gradient accumulation included."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._side.wait_event(ev)
        with torch.cuda.stream(self._side):
            b.step()
            b.done.record(self._side)
        b.fired = True

    def _on_grad(self, p) -> None:
        b = self._bucket_of[id(p)]
        b.pending -= 1
        if b.pending == 0 and not b.fired:
            self._fire(b)

    def step(self) -> None:
        """Finish this round: every bucket pushes its gradient (the module's .grad) and loads
        the weights the next gradient must be computed at."""
        if not self.pipelined:
            for b in self.buckets:
                b.step()
            return
        main = torch.cuda.current_stream(self.device)
        for b in self.buckets:
            if not b.fired:  # parameters that got no gradient this round (zero buffers)
                self._fire(b)
            main.wait_event(b.done)
            b.fired = False
            b.pending = len(b.params)

    def flush(self) -> None:
        """Apply the last round and load the global weights W into the module."""
        for b in self.buckets:
            b.worker.flush()
            b.load(b.worker.weights)

    def grad_norm(self, t: int) -> float:
        """||round-t mean gradient||_2 over every key (engine.py:521)."""
        return sum(b.worker.grad_norm(t) ** 2 for b in self.buckets) ** 0.5

    def gradient(self) -> torch.Tensor:
        """The gradient pushed in the last round (every key, registration order) — valid until
        the next backward starts accumulating (two buffers alternate)."""
        out = torch.empty(self.layout.total, dtype=torch.float32, device=self.device)
        start = {s.name: s.start for s in self.layout.spans}
        for b in self.buckets:
            g = b.grads[(b.worker.t - 1) % 2]
            for s in b.layout.spans:
                out[start[s.name]:start[s.name] + s.length].copy_(g[s.start:s.start + s.length])
        return out

    def residual(self) -> torch.Tensor:
        """fp64 residual of every key, in the module's registration (layout) order."""
        out = torch.empty(self.layout.total, dtype=torch.float64, device=self.device)
        start = {s.name: s.start for s in self.layout.spans}
        for b in self.buckets:
            r = b.worker.residual
            for s in b.layout.spans:
                out[start[s.name]:start[s.name] + s.length].copy_(r[s.start:s.start + s.length])
        return out

    def close(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []
        for b in self.buckets:
            b.worker.close()
