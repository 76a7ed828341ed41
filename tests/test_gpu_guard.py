"""Memory-safety checks of our own (compute-sanitizer is closed on this GPU pool).

* Out-of-bounds writes (memcheck's job): every buffer a kernel writes is the middle of a
  larger allocation whose guard bands are filled with a sentinel; after the kernel the
  guards must be untouched. Layouts with odd key lengths (partial last tiles, keys not
  16-B aligned) and misaligned buffer starts exercise every masked / scalar path.
* Unwritten outputs (initcheck's job): outputs are pre-filled with a sentinel that no
  kernel can produce; afterwards every element (every packed word, pad bits included)
  must have been written.
* Races (racecheck / synccheck's job): each kernel runs twice on identical inputs and
  under static vs dynamic tile scheduling; results must be bitwise identical (the
  grad-norm metric excepted: an fp64 atomic sum over CTAs, order-dependent in its last
  bits, so compared to 1e-12).
All through the public C ABI, against the oracle values where they exist.
"""

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O

pytestmark = pytest.mark.gpu
G = 1024  # guard elements on each side
SENT32 = 0x7FC0DEAD  # a NaN payload no kernel writes
SENT64 = 0x7FF8DEADBEEF0001


@pytest.fixture(scope="module")
def L():
    from paper_2106_10796_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)
    return _lib


def guarded(n, dtype, fill=None, shift=0):
    """Tensor of n elements (view) inside a buffer with G-element sentinel guards; shift
    elements of extra misalignment at the front."""
    it = torch.int64 if dtype == torch.float64 else torch.int32
    sent = SENT64 if dtype == torch.float64 else SENT32
    buf = torch.full((n + 2 * G + shift,), sent, dtype=it, device="cuda")
    view = buf[G + shift:G + shift + n].view(dtype)
    if fill is not None:
        view.copy_(torch.as_tensor(fill, device="cuda").to(dtype))
    return buf, view


def guards_intact(buf, n, shift=0):
    sent = SENT64 if buf.dtype == torch.int64 else SENT32
    h = buf.cpu().numpy()
    return bool(np.all(h[:G + shift] == sent) and np.all(h[G + shift + n:] == sent))


def all_written(view):
    h = view.contiguous().view(torch.int64 if view.dtype == torch.float64 else torch.int32).cpu().numpy()
    sent = SENT64 if view.dtype == torch.float64 else SENT32
    return bool(np.all(h != sent))


LAYOUTS = [[1], [17], [4099, 1, 33], [1000, 37, 16, 1], [513] * 7, [70_001, 3, 129]]


@pytest.mark.parametrize("shift", [0, 1, 3])
@pytest.mark.parametrize("sizes", LAYOUTS, ids=lambda s: "-".join(map(str, s))[:30])
def test_quantize_guards_and_init(L, sizes, shift):
    from paper_2106_10796_b200.layout import Layout

    lay = Layout.from_lengths(sizes)
    n, nw = lay.total, lay.n_words
    rng = np.random.default_rng(n + shift)
    g = (0.5 * rng.standard_normal(n)).astype(np.float32)
    r = 0.3 * rng.standard_normal(n)
    gb, gd = guarded(n, torch.float32, g, shift)
    rb, rd = guarded(n, torch.float64, r, shift)
    ob, od = guarded(n, torch.float64, None, shift)
    wb, wd = guarded(nw, torch.int32, None, shift)
    err = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    L.check(L.lib().cdsgd_quantize(lay.handle().ptr, gd.data_ptr(), L.F32, rd.data_ptr(), od.data_ptr(), wd.data_ptr(),
                                   0.5, err.data_ptr(), 0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for b, m in ((gb, n), (rb, n), (ob, n), (wb, nw)):
        assert guards_intact(b, m, shift)
    assert all_written(od) and all_written(wd)
    ow, orr = O.quantize_layout(r, g, 0.5, sizes)
    assert np.array_equal(wd.cpu().numpy().view(np.uint32), ow)
    assert np.array_equal(od.cpu().numpy().view(np.uint64), orr.view(np.uint64))


@pytest.mark.parametrize("wdt", ["f64", "f32"])
@pytest.mark.parametrize("nr", [1, 3])
@pytest.mark.parametrize("sizes", LAYOUTS, ids=lambda s: "-".join(map(str, s))[:30])
def test_fused_round_guards_init_and_determinism(L, sizes, nr, wdt):
    from paper_2106_10796_b200.layout import Layout

    lay = Layout.from_lengths(sizes)
    n, nw = lay.total, lay.n_words
    rng = np.random.default_rng(7 * n + nr)
    g = (0.5 * rng.standard_normal(n)).astype(np.float32)
    r = 0.3 * rng.standard_normal(n)
    w0 = rng.standard_normal(n)
    codes = np.concatenate([np.concatenate([O.pack_symbols(rng.integers(0, 3, s).astype(np.uint8)) for s in sizes])
                            for _ in range(nr)])
    wt = torch.float64 if wdt == "f64" else torch.float32
    outs = []
    for rep in range(2):
        gb, gd = guarded(n, torch.float32, g)
        rb, rd = guarded(n, torch.float64, r)
        ob, od = guarded(n, torch.float64, None)
        Wb, Wd = guarded(n, wt, w0)
        lb, ld = guarded(n, torch.float32, None)
        wb, wd = guarded(nw, torch.int32, None)
        cb, cd = guarded(nr * nw, torch.int32, codes.view(np.int32))
        err = torch.full((2,), -1, dtype=torch.int64, device="cuda")
        gn = torch.zeros(1, dtype=torch.float64, device="cuda")
        L.check(L.lib().cdsgd_fused_round(lay.handle().ptr, gd.data_ptr(), rd.data_ptr(), od.data_ptr(), L.F64,
                                          wd.data_ptr(), 0.5, err.data_ptr(), 0, Wd.data_ptr(), L.WEIGHTS[wdt],
                                          ld.data_ptr(), cd.data_ptr(), nr, nw, 0.1, 0.4, 0, gn.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        for b, m in ((gb, n), (rb, n), (ob, n), (Wb, n), (lb, n), (wb, nw), (cb, nr * nw)):
            assert guards_intact(b, m)
        assert all_written(od) and all_written(wd) and all_written(ld) and all_written(Wd)
        assert [int(x) for x in err.cpu().tolist()] == [-1, -1]
        outs.append([t.cpu().numpy().copy() for t in (od, wd, Wd, ld, gn)])
    for a, b in zip(outs[0][:4], outs[1][:4]):  # r', codes, W, loc: run to run bitwise (no races)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    # the grad-norm metric is an fp64 atomic sum over CTAs: order-dependent in the last bits
    assert abs(outs[0][4][0] - outs[1][4][0]) <= 1e-12 * max(abs(outs[0][4][0]), 1.0)
    ow, orr = O.quantize_layout(r, g, 0.5, sizes)
    assert np.array_equal(outs[0][1].view(np.uint32), ow)
    assert np.array_equal(outs[0][0].view(np.uint64), orr.view(np.uint64))


def test_engine_dynamic_vs_static_schedule_bitwise(L, tmp_path):
    """The engine's dynamically scheduled kernels (tile tickets) give bitwise the results of
    static tile ranges (CDSGD_STATIC_SCHED=1, a separate process): no schedule-dependent race."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
from oracle import cdsgd_oracle as O
from paper_2106_10796_b200.engine import HyperParams
from paper_2106_10796_b200.layout import Layout
from paper_2106_10796_b200.worker import CDSGDWorker
sizes = [300_000, 4099, 17, 70_001]
lay = Layout.from_lengths(sizes); n = lay.total
wk = CDSGDWorker(lay, HyperParams(algo="cdsgd", workers=1, k=4, warmup_n=1), O.synthetic_weights(4, n))
for t in range(10):
    wk.step(torch.from_numpy(O.synthetic_grad(4, t, 0, n)).cuda())
wk.flush()
np.savez(sys.argv[1], W=wk.weights.cpu().numpy(), r=wk.residual.cpu().numpy(), loc=wk.compute_weights().cpu().numpy())
''' % root
    res = {}
    for mode in ("dyn", "static"):
        env = dict(os.environ)
        if mode == "static":
            env["CDSGD_STATIC_SCHED"] = "1"
        out = str(tmp_path / f"{mode}.npz")
        p = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        res[mode] = np.load(out)
    for k in ("W", "r", "loc"):
        assert np.array_equal(res["dyn"][k].view(np.uint8), res["static"][k].view(np.uint8)), k
