"""GPU parity of the row-sharded solve (config C5's path) at W = 1.

Only one GPU is available to the test driver, so the sharded handle runs with a one-rank NCCL
communicator: every collective of the sharded path executes (all-gather of the Uᵀ blocks,
per-pass all-reduce of column sums and mass, δ all-reduce, N all-gather before the LAP) and the
K-blocked GEMM operand, the row-block SDSN kernels (K4s) and the row-block precondition/update
are exercised end to end.  FP64 mode is held to the oracle at ≤ 1e-9 per outer iteration with
replayed pass counts (same acceptance as the single-GPU path); mixed modes to the objective.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2508_00887_b200 as fb
from synth import config_c1, config_c2

pytestmark = pytest.mark.gpu


def _g(x, dt=torch.float64):
    return torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


def _sharded(n, **kw):
    uid = fb.fram_get_unique_id()
    return fb.fram_create_sharded(n, kw.pop("lam", 1.0), fb.Schedule(**kw), uid, rank=0, world=1)


@pytest.mark.parametrize("seed", [0, 1])
def test_sharded_w1_fp64_c1_replay(seed):
    inst = config_c1(seed)
    h = _sharded(inst.n, theta=inst.theta, flags=fb.FLAG_TRACE | fb.FLAG_CHECK_SYMMETRY)
    st, stats, X, perm = fb.fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")
    assert stats["sdsn_kernel"] == 3
    ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta, replay=stats["passes"])
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), ref["perm"])
    assert stats["outer_iters"] == len(ref["passes"])


def test_sharded_w1_fp64_c2_small_unary_replay():
    inst = config_c2(0, n=130)                       # ragged n (not a multiple of 16 / 64)
    rng = np.random.Generator(np.random.PCG64(5))
    K = rng.random((inst.n, inst.n)) * 0.1
    h = _sharded(inst.n, theta=inst.theta, lam=0.5, flags=fb.FLAG_TRACE, max_outer=6)
    st, stats, X, perm = fb.fram_solve(h, _g(inst.A), _g(inst.B), _g(K), precision="fp64")
    ref = oracle.fram(inst.A, inst.B, K, lam=0.5, theta=inst.theta, replay=stats["passes"])
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), oracle.lap_max(X.cpu().numpy()))


def test_sharded_w1_fp64_several_rows_per_cta_replay():
    # n = 437 on 148 CTAs: 2-3 rows per CTA, so the snake row order of odd passes and the per-CTA row
    # offsets are exercised (n ≤ 148 gives every CTA one row)
    inst = config_c2(2, n=437)
    h = _sharded(inst.n, theta=inst.theta, flags=fb.FLAG_TRACE, max_outer=3)
    st, stats, X, perm = fb.fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")
    ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta, max_outer=3, replay=stats["passes"])
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), oracle.lap_max(X.cpu().numpy()))


def test_sharded_w1_fp64_long_rows_closed_form():
    # n = 8200 in FP64: a row is 4100 two-element vectors, more than one 4096-vector work unit of
    # K4s (the single-GPU path stops at n = 8192 in FP64).  With A = Ã = 0 the gradient is the
    # constant λK' (K' = K/max K), so D = SDSN(λK') every iteration and closed form C
    # gives N_t = D + (1−α)^t (N_0 − D); D comes from the oracle's Alg. 2 with the same 7 passes.
    n, alpha = 8200, 0.95
    rng = np.random.Generator(np.random.PCG64(11))
    K = rng.random((n, n)) * 0.01
    K[np.diag_indices(n)] += 1.0
    Kp = K / K.max()
    D, _ = oracle.sdsn(Kp, theta=10.0, sdsn_fixed=7)
    N0 = np.full((n, n), 1.0 / n)
    want = D + (1.0 - alpha) ** 2 * (N0 - D)
    Z = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    h = _sharded(n, theta=10.0, alpha=alpha, sdsn_fixed=7, max_outer=2)
    _, stats, X, perm = fb.fram_solve(h, Z, Z, _g(K), precision="fp64")
    assert stats["passes"] == [7, 7]
    assert np.max(np.abs(X.cpu().numpy() - want)) <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), np.arange(n))


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_sharded_w1_mixed_matches_single_gpu(prec):
    inst = config_c2(1, n=256)
    hs = _sharded(inst.n, theta=inst.theta)
    _, ss, Xs, ps = fb.fram_solve(hs, _g(inst.A, torch.float32), _g(inst.B, torch.float32), precision=prec)
    h1 = fb.fram_create(inst.n, schedule=fb.Schedule(theta=inst.theta))
    _, s1, X1, p1 = fb.fram_solve(h1, _g(inst.A, torch.float32), _g(inst.B, torch.float32), precision=prec)
    phi_s = oracle.objective_perm(inst.A, inst.B, None, ps.cpu().numpy())
    phi_1 = oracle.objective_perm(inst.A, inst.B, None, p1.cpu().numpy())
    assert abs(phi_s - phi_1) <= 1e-3 * abs(phi_1)
    acc_s = oracle.node_accuracy(ps.cpu().numpy(), inst.perm_true)
    acc_1 = oracle.node_accuracy(p1.cpu().numpy(), inst.perm_true)
    assert abs(acc_s - acc_1) <= 0.005
    assert np.array_equal(ps.cpu().numpy(), oracle.lap_max(Xs.cpu().numpy()))


def test_sharded_entry_point_restrictions_and_errors():
    inst = config_c1(0)
    h = _sharded(inst.n, theta=inst.theta)
    with pytest.raises(fb.FramError) as e:
        fb.fram_lap(h, _g(np.eye(inst.n)))
    assert e.value.status == fb.FRAM_ERR_USAGE
    with pytest.raises(fb.FramError) as e:
        fb.fram_solve(h, _g(np.zeros((inst.n, inst.n))), _g(np.zeros((inst.n, inst.n))), precision="fp64")
    assert e.value.status == fb.FRAM_ERR_DATA
    hb = _sharded(100, theta=10.0)
    with pytest.raises(fb.FramError) as e:                 # mixed precision needs (n/W) % 64 == 0
        fb.fram_solve(hb, _g(np.ones((100, 100)), torch.float32), _g(np.ones((100, 100)), torch.float32),
                      precision="bf16")
    assert e.value.status == fb.FRAM_ERR_USAGE
