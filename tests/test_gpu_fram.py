"""GPU end-to-end parity of fram_solve (Alg. 1) against the FP64 oracle.

Acceptance (BASELINE.json north_star):
  FP64 mode  : max|N_gpu⁽ᵗ⁾ − N_oracle⁽ᵗ⁾| ≤ 1e-9 per outer iteration, with the oracle replaying
               the GPU's SDSN pass counts (one extra pass moves N by ~1e-4 [M14]).
  mixed modes: |Φ(M_gpu) − Φ(M_oracle)|/|Φ(M_oracle)| ≤ 1e-3 and accuracy within 0.5 pp.
  LAP        : perm_gpu == oracle.lap_max(N_gpu), bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2508_00887_b200 import (FRAM_NOT_CONVERGED, FRAM_OK, Schedule, fram_create, fram_solve,
                                   FLAG_CHECK_SYMMETRY, FLAG_TRACE, FLAG_TIME_PHASES)
from synth import config_c1, config_c2, config_c4

pytestmark = pytest.mark.gpu


def _g(x, dt=torch.float64):
    return torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


def _sched(inst, **kw):
    return Schedule(theta=inst.theta, **kw)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_fram_fp64_c1_replay_per_iteration(seed):
    inst = config_c1(seed)
    n = inst.n
    h = fram_create(n, schedule=_sched(inst))
    st, stats, X, perm = fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")
    passes = stats["passes"]
    ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta, replay=passes, keep_trace=True)
    free = oracle.fram(inst.A, inst.B, None, theta=inst.theta)
    assert free["passes"] == passes                      # free-running pass counts agree
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    for t in sorted({1, max(1, len(passes) // 2), len(passes)}):
        ht = fram_create(n, schedule=_sched(inst, replay=passes[:t]))
        _, _, Xt, _ = fram_solve(ht, _g(inst.A), _g(inst.B), precision="fp64")
        assert np.max(np.abs(Xt.cpu().numpy() - ref["Ns"][t - 1])) <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), oracle.lap_max(X.cpu().numpy()))
    assert np.array_equal(perm.cpu().numpy(), ref["perm"])
    assert st == FRAM_OK and stats["converged"]


def test_fram_fp64_c2_small_replay():
    inst = config_c2(0, n=160)
    h = fram_create(inst.n, schedule=_sched(inst))
    _, stats, X, perm = fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")
    ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta, replay=stats["passes"])
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), ref["perm"])
    assert np.max(np.abs(np.array(stats["deltas"]) - np.array(ref["deltas"]))) <= 1e-9


@pytest.mark.parametrize("prec", ["bf16", "tf32", "fp16"])
def test_fram_mixed_c2(prec):
    inst = config_c2(1, n=300)
    h = fram_create(inst.n, schedule=_sched(inst))
    st, stats, X, perm = fram_solve(h, _g(inst.A), _g(inst.B), precision=prec)
    ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta)
    p = perm.cpu().numpy()
    phi = oracle.objective_perm(inst.A, inst.B, None, p)
    phi_o = oracle.objective_perm(inst.A, inst.B, None, ref["perm"])
    assert abs(phi - phi_o) / abs(phi_o) <= 1e-3
    acc = oracle.node_accuracy(p, inst.perm_true)
    acc_o = oracle.node_accuracy(ref["perm"], inst.perm_true)
    assert abs(acc - acc_o) <= 0.005
    assert np.array_equal(p, oracle.lap_max(X.cpu().numpy()))


def test_fram_host_buffers_match_device():
    inst = config_c1(5)
    h = fram_create(inst.n, schedule=_sched(inst))
    _, s1, X1, p1 = fram_solve(h, _g(inst.A), _g(inst.B), precision="bf16")
    _, s2, X2, p2 = fram_solve(h, np.ascontiguousarray(inst.A), np.ascontiguousarray(inst.B), precision="bf16")
    assert isinstance(X2, np.ndarray)
    assert np.array_equal(X1.cpu().numpy(), X2) and np.array_equal(p1.cpu().numpy(), p2)
    assert s1["passes"] == s2["passes"]


def test_fram_not_converged_writes_outputs():
    inst = config_c1(0)
    h = fram_create(inst.n, schedule=_sched(inst, max_outer=2))
    st, stats, X, perm = fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")
    assert st == FRAM_NOT_CONVERGED and stats["outer_iters"] == 2
    ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta, max_outer=2)
    assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
    assert sorted(perm.cpu().numpy()) == list(range(inst.n))


def test_fram_unary_term_dspfp_and_x0():
    # K ≠ 0, explicit X0, λ = 0.5, and the DSPFP projection (no θ-scaling, 30 fixed passes; NEXT-1).
    rng = np.random.Generator(np.random.PCG64(9))
    inst = config_c1(7)
    n = inst.n
    K = rng.random((n, n))
    X0 = rng.random((n, n))
    X0 /= X0.sum()
    X0 *= n
    for flags, fixed in ((FLAG_CHECK_SYMMETRY | FLAG_TRACE, 0), (FLAG_CHECK_SYMMETRY | FLAG_TRACE | 4, 30)):
        h = fram_create(n, lam=0.5, schedule=Schedule(theta=10.0, flags=flags, sdsn_fixed=fixed))
        _, stats, X, perm = fram_solve(h, _g(inst.A), _g(inst.B), _g(K), _g(X0), precision="fp64")
        ref = oracle.fram(inst.A, inst.B, K, lam=0.5, theta=10.0, X0=X0, replay=stats["passes"],
                          scale=not (flags & 4))
        assert np.max(np.abs(X.cpu().numpy() - ref["N"])) <= 1e-9
        assert np.array_equal(perm.cpu().numpy(), ref["perm"])


def test_fram_c4_full_size_bf16():
    # BASELINE config C4 (n=4096, BA m=5, 5% rewiring), bf16-GEMM/fp32-SDSN, the bench's launch
    # configuration and schedule: size-independent properties of the output.  The comparison with the
    # oracle's full C4 solve is tests/test_gpu_acceptance.py.
    inst = config_c4(0)
    n = inst.n
    h = fram_create(n, schedule=_sched(inst, flags=FLAG_CHECK_SYMMETRY | FLAG_TRACE | FLAG_TIME_PHASES))
    st, stats, X, perm = fram_solve(h, _g(inst.A, torch.float32), _g(inst.B, torch.float32), precision="bf16")
    Xn = X.cpu().numpy()
    p = perm.cpu().numpy()
    assert np.all(Xn >= 0)
    # mass: every D_t has Σ/n − 1 ≤ γ of its last pass input (γ nonincreasing), and N is a
    # convex combination of N⁽⁰⁾ and the D_t; capped SDSN calls (sdsn_max = 1000) leave γ > γ_th.
    mass = Xn.sum() / n - 1
    assert -1e-9 <= mass <= max(stats["gamma_last"]) + 1e-6
    assert sorted(p) == list(range(n))
    assert stats["total_passes"] == sum(stats["passes"]) and len(stats["passes"]) == stats["outer_iters"]


@pytest.mark.parametrize("n", [1, 2, 3, 5])
@pytest.mark.parametrize("prec", ["fp64", "bf16"])
def test_fram_tiny_sizes(n, prec):
    # degenerate sizes: one node (the only permutation), two and three nodes (ragged everywhere)
    rng = np.random.Generator(np.random.PCG64(100 + n))
    A = rng.random((n, n))
    A = A + A.T
    sig = rng.permutation(n)
    B = np.empty_like(A)
    B[np.ix_(sig, sig)] = A                             # B[σ(i), σ(j)] = A[i, j] (R18)
    h = fram_create(n, schedule=Schedule(theta=10.0))
    st, stats, X, perm = fram_solve(h, _g(A), _g(B), precision=prec)
    assert st in (FRAM_OK, FRAM_NOT_CONVERGED)
    p = perm.cpu().numpy()
    assert sorted(p) == list(range(n))
    Xn = X.cpu().numpy()
    assert np.all(Xn >= 0)
    assert np.array_equal(p, oracle.lap_max(Xn))
    if prec == "fp64":
        ref = oracle.fram(A, B, None, theta=10.0, replay=stats["passes"])
        assert np.max(np.abs(Xn - ref["N"])) <= 1e-9
        assert np.array_equal(p, ref["perm"])
    if n == 1:
        assert p[0] == 0 and abs(Xn[0, 0] - 1.0) <= 1e-6


def test_fram_above_on_chip_limit_bf16():
    # n = 5000 > 4096: the FP32 SDSN streams through L2/HBM (K4) and the LAP runs on the 4-CTA cluster with
    # 8 columns per thread; a few outer iterations, output properties and the bit-exact LAP of the GPU's N
    rng = np.random.Generator(np.random.PCG64(5000))
    n = 5000
    from synth import ba_graph
    A = ba_graph(rng, n, 3)
    sig = rng.permutation(n)
    B = np.empty_like(A)
    B[np.ix_(sig, sig)] = A
    h = fram_create(n, schedule=Schedule(theta=10.0, max_outer=3, sdsn_max=50))
    st, stats, X, perm = fram_solve(h, _g(A, torch.float32), _g(B, torch.float32), precision="bf16")
    assert st in (FRAM_OK, FRAM_NOT_CONVERGED) and stats["sdsn_kernel"] == 1 and stats["passes"] == [50, 50, 50]
    Xn = X.cpu().numpy()
    assert np.all(Xn >= 0)
    p = perm.cpu().numpy()
    assert np.array_equal(p, oracle.lap_max(Xn))
