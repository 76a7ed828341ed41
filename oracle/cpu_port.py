"""CPU port of the reference CD-SGD round — TEST INFRASTRUCTURE / CPU BASELINE ONLY.

Binds oracle/_build/libcdsgd_oracle.so (the C restatement in cdsgd_oracle.c,
OpenMP over all host threads) and drives it as the reference's lock-step
scheduler would (engine.py:614-663) for synthetic gradients. Results are
bit-identical to oracle/cdsgd_oracle.py (checked in tests/test_oracle_cport.py),
which is itself pinned to the reference's golden vectors. Falls back to the NumPy
restatement (single thread) only if the C port has not been built — this is the
CPU *baseline*, never the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import time

import numpy as np

from . import cdsgd_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libcdsgd_oracle.so")

_lib = None


def load(build: bool = True):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO) and build:
        subprocess.run(["make", "-s", "-C", HERE], check=False, capture_output=True)
    if not os.path.exists(SO):
        return None
    lib = C.CDLL(SO)
    p = C.c_void_p
    lib.cdsgd_ref_threads.restype = C.c_int
    lib.cdsgd_ref_set_threads.argtypes = [C.c_int]
    lib.cdsgd_ref_quantize_layout.restype = C.c_int64
    lib.cdsgd_ref_quantize_layout.argtypes = [p, p, p, p, p, C.c_int32, C.c_double]
    lib.cdsgd_ref_aggregate_quant.restype = C.c_int64
    lib.cdsgd_ref_aggregate_quant.argtypes = [p, C.c_int32, C.c_int64, p, C.c_int32, C.c_double, p]
    lib.cdsgd_ref_aggregate_full.argtypes = [p, C.c_int32, C.c_int64, C.c_int64, p]
    lib.cdsgd_ref_global_update.argtypes = [p, p, C.c_int64, C.c_double]
    lib.cdsgd_ref_local_update.argtypes = [p, p, p, C.c_int64, C.c_double]
    lib.cdsgd_ref_pack.restype = C.c_int64
    lib.cdsgd_ref_pack.argtypes = [p, C.c_int64, p]
    lib.cdsgd_ref_unpack.argtypes = [p, C.c_int64, p]
    _lib = lib
    return lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class CPortEngine:
    """Lock-step CD-SGD (cdsgd algo, N workers) on the C port; closed-form slots.

    Same rounds as oracle.LockstepOracle (engine.py:288-663): warm-up rounds are
    full precision; formal round t compresses iff (t - warmup + 1) % k != 0; the
    compute weights of worker w for round t >= max(warmup, 1) are
    W_{t-1} - eta_l * g_{t-1,w} (engine.py:385-392)."""

    def __init__(self, w0, sizes, n_workers, k=4, alpha=0.5, eta_g=0.1, eta_l=0.4, warmup=0):
        self.lib = load()
        if self.lib is None:
            raise RuntimeError("C port not built")
        self.sizes = np.asarray(sizes, dtype=np.int64)
        self.n = int(self.sizes.sum())
        self.nw = int(((self.sizes + 15) // 16).sum())
        self.N, self.k, self.alpha, self.eta_g, self.eta_l, self.warm = n_workers, k, alpha, eta_g, eta_l, warmup
        self.W = np.asarray(w0, dtype=np.float64).copy()
        self.res = np.zeros((n_workers, self.n))
        self.words = np.zeros((n_workers, self.nw), dtype=np.uint32)
        self.mean = np.zeros(self.n)
        self.loc = np.zeros((n_workers, self.n))
        self.t = 0

    def compressed(self, t):
        return t >= self.warm and (t - self.warm + 1) % self.k != 0

    def step(self, grads: np.ndarray) -> None:
        """grads: float32 [N, n]."""
        lib = self.lib
        grads = np.ascontiguousarray(grads, dtype=np.float32)
        if self.compressed(self.t):
            for w in range(self.N):
                bad = lib.cdsgd_ref_quantize_layout(_p(self.res[w]), _p(grads[w]), _p(self.res[w]), _p(self.words[w]),
                                                    _p(self.sizes), len(self.sizes), self.alpha)
                if bad >= 0:
                    raise O.OracleNumericError("non-finite accumulated gradient", bad)
            lib.cdsgd_ref_aggregate_quant(_p(self.words), self.N, self.nw, _p(self.sizes), len(self.sizes),
                                          self.alpha, _p(self.mean))
        else:
            lib.cdsgd_ref_aggregate_full(_p(grads), self.N, self.n, self.n, _p(self.mean))
        # local update from the pulled base (engine.py:385-392; the base is W_t before this round's commit)
        if self.t >= self.warm - 1:
            for w in range(self.N):
                lib.cdsgd_ref_local_update(_p(self.W), _p(grads[w]), _p(self.loc[w]), self.n, self.eta_l)
        lib.cdsgd_ref_global_update(_p(self.W), _p(self.mean), self.n, self.eta_g)
        self.t += 1


def time_rounds(sizes, n_workers, k, alpha, rounds, seed=0, threads=None, warm=1):
    """Run `warm` untimed + `rounds` timed lock-step rounds; returns (seconds, kind, cores, impl)."""
    n = int(np.sum(sizes))
    rng = np.random.default_rng(seed)
    pool = [(0.3 * rng.standard_normal((n_workers, n))).astype(np.float32) for _ in range(2)]
    w0 = rng.standard_normal(n)
    lib = load()
    if lib is not None:
        if threads:
            lib.cdsgd_ref_set_threads(int(threads))
        eng = CPortEngine(w0, sizes, n_workers, k=k, alpha=alpha)
        for r in range(warm):  # first touch of every buffer (page faults) stays out of the timing
            eng.step(pool[r % 2])
        t0 = time.perf_counter()
        for r in range(rounds):
            eng.step(pool[(warm + r) % 2])
        secs = time.perf_counter() - t0
        cores = lib.cdsgd_ref_threads()
        return secs, "port", cores, (f"C restatement of the reference NumPy round (oracle/cdsgd_oracle.c, "
                                     f"bit-identical), OpenMP {cores} threads")
    orc = O.LockstepOracle(w0, list(sizes), O.OracleHP("cdsgd", n_workers, 0.1, 0.4, k, alpha, 0))
    for r in range(warm):
        orc.step(list(pool[r % 2]))
    t0 = time.perf_counter()
    for r in range(rounds):
        orc.step(list(pool[(warm + r) % 2]))
    return time.perf_counter() - t0, "port", 1, "NumPy restatement (oracle/cdsgd_oracle.py), 1 thread"
