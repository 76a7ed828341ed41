"""Per-round records and metrics.csv, as the reference writes them.

Mirrors ``IterationRecord`` (engine.py:147-164), ``_make_record`` (engine.py:593-611) and
the CLI's metrics.csv (cli.py:36-75): columns iter, epoch, loss, grad_norm, bytes,
compressed, wall_micros, floats written with ``repr``.

* ``bytes`` is the reference-equivalent push volume of the round summed over all workers
  (engine.py:397-407): a compressed round pushes each key's SERIALIZED payload,
  13 + 4*ceil(n_k/16) bytes (codec.py:67-69, 111-112); a full-precision round 8 bytes per
  element (fp64 vectors). It is what the reference's transport would have carried, not
  what NVLink moved (the engine ships 4*ceil(n_k/16) code bytes and fp32 corrections).
* ``grad_norm`` is ||round mean||_2 (engine.py:521), from the engine's device grad-norm
  ring. Recording never synchronises: each round's norm is copied device -> pinned host
  on the stream once the round is applied, and resolved when the records are read.
* ``wall_micros`` is 0 in the reference's deterministic in-process mode (engine.py:151-155);
  ``Recorder(wall=True)`` stores the host time between successive step() calls instead.
"""

from __future__ import annotations

import csv
import math
import time
from dataclasses import dataclass
from typing import Optional

import torch

from .codec import serialized_payload_bytes

METRICS_COLUMNS = ("iter", "epoch", "loss", "grad_norm", "bytes", "compressed", "wall_micros")  # cli.py:36
DIVERGENCE_LOSS_LIMIT = 1e6  # engine.py:78


class TrainingDiverged(RuntimeError):
    """Mirror of engine.TrainingDiverged (engine.py:86-93): non-finite or exploding loss."""

    def __init__(self, iteration: int, loss: float):
        super().__init__(f"training diverged at iteration {iteration}: loss={loss!r}")
        self.iteration = iteration
        self.loss = loss


@dataclass
class IterationRecord:
    """One committed global round (engine.py:147-164)."""

    iteration: int
    epoch: int
    train_loss: float
    grad_norm: float
    bytes_pushed: int
    compressed: bool
    wall_micros: int


def round_bytes_pushed(layout, compressed: bool, n_workers: int) -> int:
    """Reference-equivalent bytes of one round over all workers (engine.py:397-407)."""
    if compressed:
        per_worker = sum(serialized_payload_bytes(s.length) for s in layout.spans)
    else:
        per_worker = 8 * layout.total
    return n_workers * per_worker


def write_metrics_csv(path, records) -> None:
    """cli.write_metrics_csv (cli.py:39-56): same header, same formatting."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(METRICS_COLUMNS)
        for r in records:
            w.writerow([r.iteration, r.epoch, repr(r.train_loss), repr(r.grad_norm), r.bytes_pushed,
                        int(r.compressed), r.wall_micros])


def read_metrics_csv(path) -> list:
    """cli.read_metrics_csv (cli.py:59-75)."""
    out = []
    with open(path, newline="") as fh:
        rd = csv.reader(fh)
        header = next(rd)
        if tuple(header) != METRICS_COLUMNS:
            raise ValueError(f"unexpected metrics header {header}")
        for row in rd:
            out.append(IterationRecord(int(row[0]), int(row[1]), float(row[2]), float(row[3]), int(row[4]),
                                       bool(int(row[5])), int(row[6])))
    return out


class Recorder:
    """Collects one IterationRecord per round of a CDSGDWorker without host syncs.

        rec = Recorder(worker, batches_per_epoch=len(loader))
        for t, (x, y) in enumerate(loader):
            loss = ...; worker.step(g)
            rec.record(loss)                 # loss: float or 0-d CUDA tensor (read lazily)
        worker.flush(); rec.records()        # resolves grad norms / losses (one sync)

    The grad norm of round t is accumulated by the kernel that applies round t (inside
    step t+1, or flush); record() enqueues its device->host copy right after that kernel.
    """

    def __init__(self, worker, batches_per_epoch: int = 0, wall: bool = False, check_divergence: bool = True):
        if not worker.gnorm_ring or worker.gnorm_ring < 4:
            raise ValueError("Recorder needs a worker with gnorm_ring >= 4")
        self.w = worker
        self.bpe = int(batches_per_epoch)
        self.wall = wall
        self.check = check_divergence
        self._pending = []  # (t, epoch, loss, compressed, wall_us, norm_slot_index or None)
        self._host = torch.zeros(1024, dtype=torch.float64, pin_memory=True)
        self._n = 0
        self._t_last = None
        self._resolved: list = []

    def _copy_norm(self, t: int) -> int:
        if self._n == self._host.numel():
            bigger = torch.zeros(2 * self._n, dtype=torch.float64, pin_memory=True)
            torch.cuda.current_stream(self.w.device).synchronize()
            bigger[: self._n].copy_(self._host)
            self._host = bigger
        i = self._n
        self._n += 1
        self._host[i:i + 1].copy_(self.w.gnorm[t % self.w.gnorm_ring:t % self.w.gnorm_ring + 1], non_blocking=True)
        return i

    def record(self, loss=0.0) -> None:
        """Record the round just stepped (worker.t - 1). Call once after each step()."""
        t = self.w.t - 1
        now = time.perf_counter()
        wall = 0
        if self.wall:
            wall = 0 if self._t_last is None else int(round(1e6 * (now - self._t_last)))
            self._t_last = now
        epoch = t // self.bpe if self.bpe else 0
        if isinstance(loss, torch.Tensor):
            loss = loss.detach().reshape(()).to("cpu", non_blocking=True)
        self._pending.append([t, epoch, loss, self.w.round_compressed(t), wall, None])
        # round t-1 was applied inside this step: its grad norm is final now
        self._attach_norm(t - 1)

    def _attach_norm(self, t: int) -> None:
        for p in reversed(self._pending):
            if p[0] == t:
                if p[5] is None:
                    p[5] = self._copy_norm(t)
                return
            if p[0] < t:
                return

    def records(self) -> list:
        """Resolve and return every record so far (call after worker.flush() for the last round)."""
        if self._pending and self._pending[-1][5] is None and not self.w.state().pending:
            self._attach_norm(self._pending[-1][0])
        torch.cuda.current_stream(self.w.device).synchronize()
        layout, n_workers = self.w.layout, self.w.world
        keep = []
        for t, epoch, loss, comp, wall, slot in self._pending:
            if slot is None:  # round not applied yet (flush() not called)
                keep.append([t, epoch, loss, comp, wall, slot])
                continue
            loss = float(loss)
            if self.check and (not math.isfinite(loss) or loss > DIVERGENCE_LOSS_LIMIT):
                raise TrainingDiverged(t, loss)  # engine.py:609-610
            norm = math.sqrt(max(float(self._host[slot]), 0.0))
            self._resolved.append(IterationRecord(t, epoch, loss, norm, round_bytes_pushed(layout, comp, n_workers),
                                                  bool(comp), wall))
        self._pending = keep
        return list(self._resolved)
