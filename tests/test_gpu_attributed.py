"""GPU parity of fram_solve_attributed (NEXT-2/NEXT-3, reading R30): attributed graphs of unequal size,
padded to the handle's n with isolated zero-attribute nodes, K = F·F̃ᵀ computed on the device (FP64
DMMA), then Alg. 1.  FP64 mode is held to oracle.fram_attributed at ≤ 1e-9 with replayed pass counts;
mixed precision to planted-subgraph recovery."""
import numpy as np
import pytest
import torch

import oracle
import paper_2508_00887_b200 as fb

pytestmark = pytest.mark.gpu


def _g(x, dt=torch.float64):
    return torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


def _planted(seed, n2, n1, d, p=0.25):
    rng = np.random.Generator(np.random.PCG64(seed))
    B = (rng.random((n2, n2)) < p).astype(float)
    B = np.triu(B, 1)
    B = B + B.T
    Ft = np.maximum(0.0, rng.normal(size=(n2, d)))
    emb = rng.permutation(n2)[:n1]
    return B[np.ix_(emb, emb)], B, Ft[emb], Ft, emb


@pytest.mark.parametrize("m,n1,n2,d", [(30, 24, 30, 8), (40, 33, 27, 5), (64, 64, 64, 16)])
def test_attributed_fp64_replay(m, n1, n2, d):
    rng = np.random.Generator(np.random.PCG64(m + n1))
    A = rng.random((n1, n1)) * (rng.random((n1, n1)) < 0.3); A = np.triu(A, 1); A = A + A.T
    B = rng.random((n2, n2)) * (rng.random((n2, n2)) < 0.3); B = np.triu(B, 1); B = B + B.T
    F, Ft = rng.random((n1, d)), rng.random((n2, d))
    h = fb.fram_create(m, lam=0.7, schedule=fb.Schedule(theta=10.0, flags=fb.FLAG_TRACE, max_outer=15))
    st, stats, X, perm = fb.fram_solve_attributed(h, _g(A), _g(B), _g(F), _g(Ft), precision="fp64")
    ref = oracle.fram_attributed(A, B, F, Ft, m, lam=0.7, theta=10.0, replay=stats["passes"])
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), ref["perm_attr"])
    if n1 > n2:
        assert (perm.cpu().numpy() == -1).sum() == n1 - n2


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_attributed_mixed_recovers_planted_subgraph(prec):
    A, B, F, Ft, emb = _planted(77, 30, 24, 8)
    h = fb.fram_create(32, lam=1.0, schedule=fb.Schedule(theta=10.0))
    st, stats, X, perm = fb.fram_solve_attributed(h, _g(A, torch.float32), _g(B, torch.float32),
                                                  _g(F, torch.float32), _g(Ft, torch.float32), precision=prec)
    assert np.array_equal(perm.cpu().numpy(), emb)


def test_attributed_without_features_and_errors():
    rng = np.random.Generator(np.random.PCG64(3))
    A = rng.random((10, 10)); A = A + A.T
    B = rng.random((12, 12)); B = B + B.T
    h = fb.fram_create(12, schedule=fb.Schedule(theta=10.0, flags=fb.FLAG_TRACE, max_outer=5))
    st, stats, X, perm = fb.fram_solve_attributed(h, _g(A), _g(B), precision="fp64")
    ref = oracle.fram_attributed(A, B, None, None, 12, theta=10.0, replay=stats["passes"])
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    with pytest.raises(fb.FramError) as e:                       # n1 > handle n
        fb.fram_solve_attributed(fb.fram_create(8), _g(A), _g(B), precision="fp64")
    assert e.value.status == fb.FRAM_ERR_USAGE
    with pytest.raises(fb.FramError) as e:                       # K = F F̃ᵀ must be ≥ 0
        fb.fram_solve_attributed(h, _g(A), _g(B), _g(-np.ones((10, 2))), _g(np.ones((12, 2))), precision="fp64")
    assert e.value.status == fb.FRAM_ERR_DATA
