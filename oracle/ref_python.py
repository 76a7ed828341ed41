"""Times the UNMODIFIED reference (cdsgd 0.1.0, pure Python/NumPy) — CPU BASELINE ONLY.

Test/measurement infrastructure: only bench.py's `cpu_baseline` / `--impl reference`
legs run this, in a subprocess, never the product path. The reference is imported from
its pip install in ``baseline/_ref`` (``python -m pip install --no-index
--no-build-isolation --no-deps --find-links /opt/wheelhouse --target baseline/_ref
<copy of /root/reference/pkg>``), which travels to the GPU box with the
repo snapshot; nothing here reads /root/reference.

Two measurements, both through the reference's own code:

* ``lockstep`` — the step oracle recipe of SURVEY §8c: Worker / ServerNode /
  _run_lockstep (engine.py:288-663) run unmodified; only ``engine.loss_and_grad``
  (engine.py:363) is replaced by a function returning pre-drawn synthetic gradients.
  Rate = N * n * rounds / seconds over rounds 1.. (round 0, first touch, excluded).
* ``bench_codec`` — ``python -m cdsgd.cli bench-codec --n N --reps R`` (cli.py:250-279),
  the reference's own codec timing harness; its printed encode / decode elements/s.

    python -m oracle.ref_python lockstep --layout resnet50 --workers 1 --rounds 6 --k 4
    python -m oracle.ref_python bench_codec --n 16384 --reps 50
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import re
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_SITE = os.path.join(ROOT, "baseline", "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SITE, "cdsgd"))


def host_info() -> dict:
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "usable_cpus": usable}


def _env():
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1",
               MKL_NUM_THREADS="1")
    env["PYTHONPATH"] = REF_SITE + os.pathsep + ROOT
    return env


def lockstep(sizes, n_workers: int, rounds: int, k: int, alpha: float = 0.5, seed: int = 0) -> dict:
    """Runs in a subprocess with baseline/_ref first on sys.path."""
    import numpy as np

    import cdsgd
    import cdsgd.engine as engine
    from cdsgd.numcore import Dataset, KeyedVector, Layout, ModelSpec

    assert os.path.realpath(cdsgd.__file__).startswith(os.path.realpath(REF_SITE)), cdsgd.__file__
    layout = Layout([(f"k{i}", int(s)) for i, s in enumerate(sizes)])
    n = layout.total
    rng = np.random.default_rng(seed)
    pool = [[(0.3 * rng.standard_normal(n)).astype(np.float32).astype(np.float64) for _ in range(n_workers)]
            for _ in range(2)]
    w0 = rng.standard_normal(n)
    calls = {"c": 0}
    stamps = []

    def fake_loss_and_grad(model, weights, X, y):  # replaces engine.py:363's gradient source only
        t, w = divmod(calls["c"], n_workers)
        calls["c"] += 1
        if w == 0:
            stamps.append(time.perf_counter())
        return 0.0, KeyedVector(pool[t % 2][w], layout)

    engine.loss_and_grad = fake_loss_and_grad
    hp = engine.HyperParams(algo="cdsgd", workers=n_workers, eta_global=0.1, eta_local=0.4, k=k, alpha=alpha,
                            warmup_n=0, batch_size=1, iters=rounds, seed=seed).validate()
    init = KeyedVector(w0.copy(), layout)
    server = engine.ServerNode(init, hp)
    ds = Dataset(np.zeros((n_workers, 1)), np.zeros(n_workers)).with_shards(n_workers)
    workers = [engine.Worker(w, ModelSpec("linear-regression", 1, 1), ds, hp, init, np.random.default_rng(w))
               for w in range(n_workers)]
    t0 = time.perf_counter()
    engine._run_lockstep(server, workers, rounds, layout)
    t1 = time.perf_counter()
    timed = rounds - 1 if rounds > 1 else 1
    start = stamps[1] if rounds > 1 else t0
    secs = t1 - start
    return {"value": n_workers * n * timed / secs / 1e9, "unit": "Gelem/s", "seconds": secs, "rounds_timed": timed,
            "rounds_run": rounds, "elements": n, "keys": len(sizes), "workers": n_workers, "k": k,
            "ms_per_round": 1e3 * secs / timed, "cores": 1,
            "how": "unmodified reference Worker/ServerNode/_run_lockstep (engine.py:288-663), synthetic "
                   "gradients via engine.loss_and_grad only (SURVEY §8c), round 0 excluded; single thread "
                   "(NumPy ufuncs), OPENBLAS_NUM_THREADS=1"}


def run_lockstep(sizes, n_workers, rounds, k, alpha=0.5, timeout=600) -> dict:
    """Subprocess wrapper (keeps the reference package out of the caller's interpreter)."""
    if not available():
        return {"unavailable": "reference not installed in baseline/_ref"}
    cmd = [sys.executable, "-m", "oracle.ref_python", "lockstep", "--sizes", ",".join(str(int(s)) for s in sizes),
           "--workers", str(n_workers), "--rounds", str(rounds), "--k", str(k), "--alpha", str(alpha)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=_env(), cwd=ROOT, timeout=timeout)
    if res.returncode != 0:
        return {"error": (res.stdout + res.stderr)[-400:]}
    return json.loads(res.stdout.strip().splitlines()[-1])


def run_bench_codec(n: int, reps: int, timeout=600) -> dict:
    """`python -m cdsgd.cli bench-codec` (cli.py:250-279), unmodified; parses its output."""
    if not available():
        return {"unavailable": "reference not installed in baseline/_ref"}
    cmd = [sys.executable, "-m", "cdsgd.cli", "bench-codec", "--n", str(n), "--reps", str(reps)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=_env(), cwd=ROOT, timeout=timeout)
    if res.returncode != 0:
        return {"error": (res.stdout + res.stderr)[-400:]}
    out = {"n": n, "reps": reps, "cores": 1, "cmd": "python -m cdsgd.cli bench-codec --n %d --reps %d" % (n, reps)}
    for key in ("encode", "decode"):
        m = re.search(rf"{key}: ([0-9.eE+]+) elements/s", res.stdout)
        out[f"{key}_elem_per_s"] = float(m.group(1)) if m else None
    return out


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("lockstep")
    a.add_argument("--sizes", default=None)
    a.add_argument("--layout", default=None)
    a.add_argument("--workers", type=int, default=1)
    a.add_argument("--rounds", type=int, default=6)
    a.add_argument("--k", type=int, default=4)
    a.add_argument("--alpha", type=float, default=0.5)
    b = sub.add_parser("bench_codec")
    b.add_argument("--n", type=int, default=16384)
    b.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    if args.cmd == "lockstep":
        if args.sizes:
            sizes = [int(s) for s in args.sizes.split(",")]
        else:
            sys.path.insert(0, ROOT)
            from paper_2106_10796_b200.layout import by_name

            sizes = by_name(args.layout).lengths
        if os.environ.get("PYTHONPATH", "").split(os.pathsep)[0] != REF_SITE:
            print(json.dumps(run_lockstep(sizes, args.workers, args.rounds, args.k, args.alpha)))
        else:
            print(json.dumps(lockstep(sizes, args.workers, args.rounds, args.k, args.alpha)))
    else:
        print(json.dumps(run_bench_codec(args.n, args.reps)))


if __name__ == "__main__":
    main()
