"""Maximum sizes: a layout of more than 2^31 elements (beyond 32-bit indexing), exact mode.

Every CD-SGD operation is elementwise per key except the 2-bit packing, which depends only
on the 16 elements of a word (codec.py:140-151). So windows of elements (16-aligned inside a
key) can be replayed independently: the C restatement of the reference round runs each
window as its own key, and the engine's residual, codes, compute weights and fp64 W must
match it bit for bit there — at the start of the vector, around element 2^31 and at the
small keys after it (element offsets > 2^31, word offsets > 2^27).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


def test_engine_beyond_2pow31_elements():
    from oracle import cpu_port
    from paper_2106_10796_b200 import _lib
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.layout import Layout
    from paper_2106_10796_b200.worker import CDSGDWorker

    _lib.load()
    torch.cuda.set_device(0)
    if cpu_port.load() is None:
        pytest.skip("C port not built")
    free, _ = torch.cuda.mem_get_info()
    big = (1 << 31) + 4096
    sizes = [big, 5000, 17]
    if free < 100 * (1 << 30):
        pytest.skip("needs ~100 GB of free device memory")
    layout = Layout.from_lengths(sizes)
    n = layout.total
    # windows: (start element, length) — 16-aligned inside key 0, whole small keys after it
    wins = [(0, 4096), ((1 << 30) + 512, 4096), ((1 << 31) - 2048, 4096 + 2048), (big, 5000), (big + 5000, 17)]
    gen = torch.Generator(device="cuda").manual_seed(31)
    w0 = torch.randn(n, device="cuda", generator=gen)
    hp = HyperParams(algo="cdsgd", workers=1, eta_global=0.1, eta_local=0.4, k=4, alpha=0.5, warmup_n=1)
    wk = CDSGDWorker(layout, hp, w0, gnorm_ring=8)
    win_lens = [ln for _, ln in wins]
    port = cpu_port.CPortEngine(torch.cat([w0[a:a + ln] for a, ln in wins]).double().cpu().numpy(), win_lens, 1, k=4,
                                alpha=0.5, eta_g=0.1, eta_l=0.4, warmup=1)
    eoff = [0]
    for s in sizes:
        eoff.append(eoff[-1] + s)
    woff = [0]
    for s in sizes:
        woff.append(woff[-1] + (s + 15) // 16)
    for t in range(6):
        g = 0.3 * torch.randn(n, device="cuda", generator=gen)
        gw = torch.cat([g[a:a + ln] for a, ln in wins]).cpu().numpy()
        wk.step(g)
        port.step(gw[None, :])
        del g
        res = torch.cat([wk.residual[a:a + ln] for a, ln in wins]).cpu().numpy()
        assert np.array_equal(res.view(np.uint64), port.res[0].view(np.uint64)), f"residual round {t}"
        if port.compressed(t):
            words = wk.gathered[t % 2].view(torch.int32)
            got, pw, o = [], [], 0
            for (a, ln) in wins:
                key = max(i for i in range(len(sizes)) if eoff[i] <= a)
                w_a = woff[key] + (a - eoff[key]) // 16
                nwin = (ln + 15) // 16
                got.append(words[w_a:w_a + nwin].cpu().numpy().view(np.uint32))
            mine = np.concatenate(got)
            assert np.array_equal(mine, port.words[0]), f"codes round {t}"
        cw = torch.cat([wk.compute_weights()[a:a + ln] for a, ln in wins]).cpu().numpy()
        # compute weights of round t+1 (>= warmup_n): loc_{t+1} = W_t - eta_l*g_t, fl32 of the reference's
        assert np.array_equal(cw.view(np.uint32), port.loc[0].astype(np.float32).view(np.uint32)), f"loc round {t}"
        np.testing.assert_allclose(cw, port.loc[0], rtol=RTOL, atol=ATOL, err_msg=f"compute weights round {t}")
    wk.flush()
    W = torch.cat([wk.weights[a:a + ln] for a, ln in wins]).cpu().numpy()
    assert W.dtype == np.float64 and np.array_equal(W.view(np.uint64), port.W.view(np.uint64)), "fp64 W not bitwise"
    wk.check()
    wk.close()
