"""Bucketed, pipelined CDSGDModule (layer-wise exchange during backward).

* buckets = 3, pipelined (post-accumulate-grad hooks, side stream) and the unbucketed module
  each against the lock-step oracle replaying the gradients autograd produced for THEM
  (residual bitwise every round, compute weights / W in tolerance; fp64 weights: bitwise):
  the reference treats every key independently (engine.py:397-402, 509-514). (Two module
  copies are not compared with each other: cuDNN's conv backward is not bitwise
  deterministic run to run.)
* memory_order="reference" on a channels_last conv net: a round's payload words are the
  oracle's for the reference's (contiguous) flatten order of each parameter."""

import numpy as np
import pytest
import torch

from oracle import cdsgd_oracle as O

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-5, 1e-6


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def net(seed):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3, padding=1), torch.nn.ReLU(), torch.nn.Conv2d(8, 8, 3),
                               torch.nn.ReLU(), torch.nn.Flatten(), torch.nn.Linear(8 * 6 * 6, 33), torch.nn.Tanh(),
                               torch.nn.Linear(33, 5)).cuda()


def flat_params(m):
    return torch.cat([p.detach().reshape(-1) for p in m.parameters()]).cpu().numpy()


@pytest.mark.parametrize("weights", ["f64", "f32"])
@pytest.mark.parametrize("buckets", [1, 3])
def test_bucketed_pipelined_module_vs_oracle(weights, buckets):
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.model import CDSGDModule

    hp = HyperParams(algo="cdsgd", workers=1, eta_global=0.05, eta_local=0.2, k=3, alpha=0.05, warmup_n=2)
    a = net(0)
    m = CDSGDModule(a, hp, buckets=buckets, weights=weights)
    assert len(m.buckets) == buckets and m.pipelined == (buckets > 1)
    sizes = m.layout.lengths
    orc = O.LockstepOracle(flat_params(a).astype(np.float64), sizes, O.OracleHP("cdsgd", 1, 0.05, 0.2, 3, 0.05, 2))
    x = torch.randn(64, 3, 8, 8, device="cuda")
    y = torch.randint(0, 5, (64,), device="cuda")
    for t in range(10):
        cw = flat_params(a)
        np.testing.assert_allclose(cw, orc.compute_weights(0), rtol=RTOL, atol=ATOL, err_msg=f"round {t}")
        if weights == "f64":  # the reference's compute weights rounded once to fp32
            assert np.array_equal(cw.view(np.uint32), orc.compute_weights(0).astype(np.float32).view(np.uint32)), t
        torch.nn.functional.cross_entropy(a(x[t * 6:t * 6 + 6]), y[t * 6:t * 6 + 6]).backward()
        m.step()
        orc.step([m.gradient().cpu().numpy()])
        assert np.array_equal(bits(m.residual().cpu().numpy()), bits(orc.workers[0].residual)), t
    m.flush()
    np.testing.assert_allclose(flat_params(a), orc.W, rtol=RTOL, atol=ATOL)
    if weights == "f64":
        assert np.array_equal(flat_params(a).view(np.uint32), orc.W.astype(np.float32).view(np.uint32))
    for t in range(1, 9):
        assert abs(m.grad_norm(t) - orc.grad_norms[t]) <= 1e-6 * max(1.0, orc.grad_norms[t])
    m.close()


def test_channels_last_reference_element_order():
    from paper_2106_10796_b200.engine import HyperParams
    from paper_2106_10796_b200.model import CDSGDModule

    a = net(1).to(memory_format=torch.channels_last)
    hp = HyperParams(algo="cdsgd", workers=1, eta_global=0.05, eta_local=0.2, k=4, alpha=0.05, warmup_n=0)
    m = CDSGDModule(a, hp)  # memory_order="reference"
    sizes = m.layout.lengths
    w0 = torch.cat([p.detach().contiguous().reshape(-1) for p in a.parameters()]).double().cpu().numpy()
    orc = O.LockstepOracle(w0, sizes, O.OracleHP("cdsgd", 1, 0.05, 0.2, 4, 0.05, 0))
    x = torch.randn(6, 3, 8, 8, device="cuda").to(memory_format=torch.channels_last)
    torch.nn.functional.cross_entropy(a(x), torch.arange(6, device="cuda") % 5).backward()
    g = torch.cat([p.grad.contiguous().reshape(-1) for p in a.parameters()]).cpu().numpy()
    m.step()
    orc.step([g])
    got = np.concatenate([p.words.cpu().numpy() for p in m.worker.round_payloads(0)])
    assert np.array_equal(got, orc.words[(0, 0)])
    m.close()
