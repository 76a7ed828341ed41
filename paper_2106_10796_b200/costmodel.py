"""Per-iteration time model of the four algorithms (paper Eq. 6-9), for calibration.

Restates the reference's closed-form model (pkg/src/cdsgd/costmodel.py:1-152, PAPER.md
eqs. 6-9) with the same names, argument meanings and errors, so timing constants
measured on B200 (scripts/calibrate_costmodel.py) can be fed to it:

    tau    compute (forward + backward) per iteration
    phi    full-precision communication per iteration
    psi    compressed communication per iteration
    delta  compression overhead per iteration
    k      correction period: iterations i with i % k == 0 ship full precision

Overlapped algorithms (local update) take max(compute, communication); ties go to
the communication branch (costmodel.py:76-80).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

REGIME_COMPUTE = "compute-bound"
REGIME_MIXED = "comm-bound-compressed"
REGIME_COMM = "comm-bound-always"
ALGOS = ("ssgd", "lusgd", "bitsgd", "cdsgd")


@dataclass(frozen=True)
class CostParams:
    """Timing constants (seconds) and the correction period (costmodel.py:29-48)."""

    tau: float
    phi: float
    psi: float
    delta: float
    k: int

    def __post_init__(self):
        for field in ("tau", "phi", "psi", "delta"):
            if getattr(self, field) < 0:
                raise ValueError(f"{field} must be >= 0")
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.psi > self.phi:
            warnings.warn(f"compressed communication ({self.psi}) slower than uncompressed ({self.phi})",
                          stacklevel=2)

    @property
    def compressed_comm(self) -> float:
        return self.delta + self.psi


def t_ssgd(p: CostParams) -> float:
    """S-SGD: compute, then full-precision communication (costmodel.py:51-53)."""
    return p.tau + p.phi


def t_loc(p: CostParams) -> float:
    """Local update: communication hidden behind compute (costmodel.py:56-58)."""
    return max(p.tau, p.phi)


def t_bit(p: CostParams) -> float:
    """BIT-SGD: compute, compression, compressed communication (costmodel.py:61-63)."""
    return p.tau + p.delta + p.psi


def comm_cd(i: int, p: CostParams) -> float:
    """Eq. 6: CD-SGD communication of 1-based iteration i (costmodel.py:66-72)."""
    if i < 1:
        raise ValueError("iteration index is 1-based")
    return p.phi if i % p.k == 0 else p.compressed_comm


def t_cd(i: int, p: CostParams) -> float:
    """Eq. 7: CD-SGD iteration time (costmodel.py:75-78); a tie is communication-bound."""
    c = comm_cd(i, p)
    return p.tau if p.tau > c else c


def avg_cd(p: CostParams) -> float:
    """Mean CD-SGD iteration over one k-period (costmodel.py:81-87)."""
    return sum(t_cd(i, p) for i in range(1, p.k + 1)) / p.k


def saving_vs_loc(i: int, p: CostParams) -> float:
    """Eq. 9, the four cases of T_s^loc (costmodel.py:90-103)."""
    c = comm_cd(i, p)
    if p.tau >= c:
        return 0.0 if p.tau >= p.phi else p.phi - p.tau
    return p.phi - p.compressed_comm if i % p.k else 0.0


def saving_vs_bit(i: int, p: CostParams) -> float:
    """Eq. 8, the three cases of T_s^bit (costmodel.py:106-118)."""
    if p.tau >= comm_cd(i, p):
        return p.compressed_comm
    return p.tau if i % p.k else p.tau + p.compressed_comm - p.phi


def classify_regime(p: CostParams) -> str:
    """Which iterations are communication-bound (costmodel.py:121-135)."""
    bound_full, bound_comp = p.tau < p.phi, p.tau < p.compressed_comm
    if not bound_full and not bound_comp:
        return REGIME_COMPUTE
    if bound_full and bound_comp:
        return REGIME_COMM
    return REGIME_MIXED


def iteration_time(algo: str, i: int, p: CostParams) -> float:
    if algo == "ssgd":
        return t_ssgd(p)
    if algo == "lusgd":
        return t_loc(p)
    if algo == "bitsgd":
        return t_bit(p)
    if algo == "cdsgd":
        return t_cd(i, p)
    raise ValueError(f"unknown algo {algo!r}")


def timeline(p: CostParams, horizon: int) -> list[tuple[int, str, float, float]]:
    """(iteration, algo, time, cumulative) rows, algorithms interleaved per iteration
    in the order ssgd, lusgd, bitsgd, cdsgd (costmodel.py:138-152)."""
    if horizon < 1:
        raise ValueError("horizon must be >= 1")
    cum = dict.fromkeys(ALGOS, 0.0)
    rows = []
    for i in range(1, horizon + 1):
        for algo in ALGOS:
            dt = iteration_time(algo, i, p)
            cum[algo] += dt
            rows.append((i, algo, dt, cum[algo]))
    return rows


def averages(p: CostParams) -> dict[str, float]:
    """Mean iteration time per algorithm (what `cdsgd costmodel` prints, cli.py:219-231)."""
    return {"ssgd": t_ssgd(p), "lusgd": t_loc(p), "bitsgd": t_bit(p), "cdsgd": avg_cd(p)}
