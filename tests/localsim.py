"""N CD-SGD workers simulated on ONE GPU through the C ABI (test infrastructure).

The analogue of the reference's lock-step scheduler (engine.py:614-663): each
simulated worker w owns its residual ping-pong, its compute weights loc_w and its own
replica W_w of the global weights (the replicated parameter server of the multi-GPU
engine); all workers' packed codes of a round land in one gathered buffer (the
all-gather), and a correction round's gradients are summed in fp32 (the all-reduce).
Per round the driver issues exactly the kernels the engine issues (cdsgd_b200.cu,
cdsgd_engine_step), through their public C entry points:

  compressed, previous round compressed : F   cdsgd_fused_round (apply(t-1) + quantize(t))
  compressed, nothing pending           : F   cdsgd_fused_round, local-only (gathered = NULL)
  compressed, previous round full       : K1  cdsgd_quantize, then K3 cdsgd_apply_full(t-1)
  correction, previous round compressed : K2  cdsgd_apply_quant(t-1) with g_next / loc
  correction, previous round full       : K3  cdsgd_apply_full(t-1) with g_next / loc
  correction, nothing pending           : local update (first local round)
  synchronous (warm-up / non-local)     : K1 + K2 or K3 applied at once, compute at W

with the reference's closed form loc_{t+1} = W_t - eta_l * g_t (engine.py:385-392).
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2106_10796_b200 import _lib

ALGOS = ("ssgd", "lusgd", "bitsgd", "cdsgd")


class LocalSim:
    def __init__(self, layout, n_workers, w0, *, algo="cdsgd", k=4, alpha=0.5, eta_g=0.1, eta_l=0.4, warmup=0,
                 fused=True, weights="f64"):
        self.lib = _lib.lib()
        self.layout, self.N, self.k, self.alpha = layout, n_workers, k, alpha
        self.eta_g, self.eta_l, self.warm, self.algo = eta_g, eta_l, warmup, algo
        self.uses_local = algo in ("lusgd", "cdsgd")
        self.n_warm = warmup if self.uses_local else 0
        self.fused = fused
        n, nw = layout.total, layout.n_words
        self.n, self.nw = n, nw
        self.lay = layout.handle().ptr
        dev = torch.device("cuda")
        self.wdt = _lib.WEIGHTS[weights]
        wt = torch.float64 if weights == "f64" else torch.float32
        w0 = torch.as_tensor(np.asarray(w0), device=dev)
        self.W = [w0.to(wt).clone() for _ in range(n_workers)]
        self.loc = [w0.to(torch.float32).clone() for _ in range(n_workers)]
        self.res = [[torch.zeros(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.float64, device=dev)]
                    for _ in range(n_workers)]
        self.rcur = [0] * n_workers
        self.gathered = [torch.zeros(n_workers * nw, dtype=torch.int32, device=dev).view(torch.uint32)
                         for _ in range(2)]
        self.gsum = [None, None]
        self.err = [torch.full((2,), -1, dtype=torch.int64, device=dev) for _ in range(n_workers)]
        self.gnorm = torch.zeros(1, dtype=torch.float64, device=dev)
        self.t = 0
        self.pending = None  # (round, compressed, grads)
        self.compute_is_loc = self.uses_local and self.n_warm == 0
        self.kernels = []  # kernel classes issued, per round
        self.gnorm_round = None  # round whose mean's sum of squares self.gnorm holds after step()

    # ------------------------------------------------------------------ schedule
    def compressed(self, t: int) -> bool:
        """Worker._push_compressed + should_compress (engine.py:217-223, 345-355)."""
        if self.uses_local and t < self.n_warm:
            return False
        if self.algo == "bitsgd":
            return True
        if self.algo == "cdsgd":
            return (t - self.n_warm + 1) % self.k != 0
        return False

    def residual(self, w):
        return self.res[w][self.rcur[w]]

    def compute_weights(self, w):
        return self.loc[w] if self.compute_is_loc else self.W[w]

    def words(self, t, w):
        """Worker w's packed codes of compressed round t (valid for the last two rounds)."""
        return self.gathered[t & 1][w * self.nw:(w + 1) * self.nw]

    # ------------------------------------------------------------------ kernels
    def _st(self):
        return torch.cuda.current_stream().cuda_stream

    def _quantize(self, w, g, slot):
        r = self.res[w]
        c = self.rcur[w]
        _lib.check(self.lib.cdsgd_quantize(self.lay, g.data_ptr(), _lib.F32, r[c].data_ptr(), r[c ^ 1].data_ptr(),
                                           slot.data_ptr() + 4 * w * self.nw, self.alpha, self.err[w].data_ptr(), 0,
                                           self._st()), "quantize")
        self.rcur[w] ^= 1

    def _fused(self, w, g, slot, gathered, gnorm):
        r = self.res[w]
        c = self.rcur[w]
        _lib.check(self.lib.cdsgd_fused_round(
            self.lay, g.data_ptr(), r[c].data_ptr(), r[c ^ 1].data_ptr(), _lib.F64, slot.data_ptr() + 4 * w * self.nw,
            self.alpha, self.err[w].data_ptr(), 0, self.W[w].data_ptr(), self.wdt, self.loc[w].data_ptr(),
            gathered.data_ptr() if gathered is not None else None, self.N, self.nw, self.eta_g, self.eta_l, 0,
            gnorm.data_ptr() if gnorm is not None else None, self._st()), "fused_round")
        self.rcur[w] ^= 1

    def _apply(self, w, p, comp, gnext, gnorm):
        loc = self.loc[w].data_ptr() if gnext is not None else None
        gp = gnext.data_ptr() if gnext is not None else None
        gn = gnorm.data_ptr() if gnorm is not None else None
        if comp:
            _lib.check(self.lib.cdsgd_apply_quant(self.lay, self.W[w].data_ptr(), self.wdt,
                                                  self.gathered[p & 1].data_ptr(),
                                                  self.N, self.nw, self.alpha, self.eta_g, gp, loc, self.eta_l,
                                                  self.err[w].data_ptr(), 0, gn, self._st()), "apply_quant")
        else:
            _lib.check(self.lib.cdsgd_apply_full(self.W[w].data_ptr(), self.wdt, self.gsum[p & 1].data_ptr(), self.N,
                                                 self.n,
                                                 self.eta_g, gp, loc, self.eta_l, None, 0, gn, self._st()),
                       "apply_full")

    # ------------------------------------------------------------------ one round of every worker
    def step(self, grads) -> None:
        """grads: list of N contiguous fp32 CUDA tensors (g_{t,w})."""
        t = self.t
        comp = self.compressed(t)
        sync = (not self.uses_local) or t < self.n_warm - 1
        slot = self.gathered[t & 1]
        gn = self.gnorm if self.N >= 1 else None
        kinds = []
        if not comp:  # the "all-reduce" of this round's gradients (fp32, identical on every replica)
            self.gsum[t & 1] = torch.stack(list(grads)).sum(0)
        pend = self.pending
        self.gnorm.zero_()
        if sync:
            if comp:
                for w in range(self.N):
                    self._quantize(w, grads[w], slot)
                kinds.append("K1")
            for w in range(self.N):
                self._apply(w, t, comp, None, gn if w == 0 else None)
            kinds.append("K2" if comp else "K3")
            self.compute_is_loc = False
        else:
            if comp and self.fused and (pend is None or pend[1]):
                for w in range(self.N):
                    self._fused(w, grads[w], slot, self.gathered[pend[0] & 1] if pend is not None else None,
                                gn if w == 0 else None)
                kinds.append("F" if pend is not None else "F_L")
            else:
                if comp:
                    for w in range(self.N):
                        self._quantize(w, grads[w], slot)
                    kinds.append("K1")
                if pend is not None:
                    for w in range(self.N):
                        self._apply(w, pend[0], pend[1], grads[w], gn if w == 0 else None)
                    kinds.append("K2" if pend[1] else "K3")
                else:
                    for w in range(self.N):
                        _lib.check(self.lib.cdsgd_local_update(self.W[w].data_ptr(), self.wdt, grads[w].data_ptr(),
                                                               _lib.F32, self.loc[w].data_ptr(), _lib.F32, self.n,
                                                               self.eta_l, self._st()), "local_update")
                    kinds.append("LU")
            self.pending = (t, comp)
            self.compute_is_loc = True
        self.kernels.append(kinds)
        self.gnorm_round = t if sync else (pend[0] if pend is not None else None)
        self.t = t + 1

    def flush(self) -> None:
        if self.pending is not None:
            p, comp = self.pending
            for w in range(self.N):
                self._apply(w, p, comp, None, None)
            self.pending = None

    def errors(self):
        return [[int(x) for x in e.cpu().tolist()] for e in self.err]
