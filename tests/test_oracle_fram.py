"""Pins for the oracle's FRAM loop (Alg. 1), preconditioning and gradient."""
import numpy as np
import pytest

import oracle
from oracle.exact import qap_brute_force
from synth import ba_graph, config_c1, er_graph


def _sym(rng, n, p=0.5):
    return er_graph(rng, n, p, weighted=True)


def test_precondition_identity(rng):
    # (A'NÃ' + λK') = (ANÃ + λK)/c; c=1 ⇒ unchanged.
    n = 9
    A, B, K = 4 * _sym(rng, n), 2 * _sym(rng, n), rng.random((n, n)) * 7
    Ap, Bp, Kp, c = oracle.precondition(A, B, K)
    assert c == max(A.max(), B.max(), K.max())
    N = rng.random((n, n))
    lhs = oracle.gradient(Ap, N, Bp, Kp, 0.7)
    rhs = (A @ N @ B + 0.7 * K) / c
    assert np.max(np.abs(lhs - rhs)) <= 1e-14 * np.abs(rhs).max()
    A1 = (rng.random((n, n)) < 0.3).astype(float)
    A1 = np.maximum(A1, A1.T)
    Ap1, Bp1, Kp1, c1 = oracle.precondition(A1, A1, None)
    assert c1 == 1.0 and np.array_equal(Ap1, A1) and np.array_equal(Bp1, A1) and np.all(Kp1 == 0)


def test_precondition_errors():
    with pytest.raises(oracle.DataError):
        oracle.precondition(np.zeros((3, 3)), np.zeros((3, 3)), None)
    with pytest.raises(oracle.DataError):
        oracle.precondition(-np.eye(3), np.eye(3), None)
    bad = np.eye(3)
    bad[0, 1] = np.nan
    with pytest.raises(oracle.DataError):
        oracle.precondition(bad, np.eye(3), None)


def test_gradient_triple_loop(rng):
    # Asymmetric operands so a transposed operand fails: G_ij = Σ_kl A_ik N_kl B_lj + λK_ij.
    n = 7
    A, N, B, K = (rng.normal(size=(n, n)) for _ in range(4))
    G = oracle.gradient(A, N, B, K, 0.3)
    ref = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            s = 0.0
            for k in range(n):
                for l in range(n):
                    s += A[i, k] * N[k, l] * B[l, j]
            ref[i, j] = s + 0.3 * K[i, j]
    assert np.max(np.abs(G - ref)) <= 1e-12
    I = np.eye(n)
    assert np.max(np.abs(oracle.gradient(I, N, I, K, 2.0) - (N + 2.0 * K))) <= 1e-15


def test_gradient_is_gradient_of_objective(rng):
    # Eq.(3): ∇Φ(N) = A N Ã + λK for symmetric A, Ã (Eq.(1)) — central differences.
    n = 6
    A, B = _sym(rng, n), _sym(rng, n)
    K = rng.random((n, n))
    N = rng.random((n, n))
    G = oracle.gradient(A, N, B, K, 0.5)
    h = 1e-6
    for i, j in [(0, 0), (1, 3), (5, 2), (4, 4)]:
        E = np.zeros((n, n))
        E[i, j] = h
        fd = (oracle.objective(A, B, K, N + E, 0.5) - oracle.objective(A, B, K, N - E, 0.5)) / (2 * h)
        assert abs(fd - G[i, j]) <= 1e-7


def test_closed_form_C(rng):
    # A = Ã = 0: D = SDSN(K') constant; N_t = D + (1−α)^t (N0 − D);
    # δ_t = α(1−α)^{t−1}‖N0−D‖/‖N_t‖   ([M15]).
    n, alpha = 8, 0.95
    K = rng.random((n, n))
    Z = np.zeros((n, n))
    out = oracle.fram(Z, Z, K, lam=1.0, theta=10.0, alpha=alpha, max_outer=5, delta_th=0.0,
                      keep_trace=True)
    Kp = K / K.max()
    D, _ = oracle.sdsn(Kp, 10.0)
    N0 = np.full((n, n), 1.0 / n)
    for t, Nt in enumerate(out["Ns"], start=1):
        ref = D + (1 - alpha) ** t * (N0 - D)
        assert np.max(np.abs(Nt - ref)) <= 1e-15
        dref = alpha * (1 - alpha) ** (t - 1) * np.linalg.norm(N0 - D) / np.linalg.norm(ref)
        assert abs(out["deltas"][t - 1] - dref) <= 1e-15 * max(1.0, dref) + 1e-16


def test_fram_scale_invariance_bitexact(rng):
    # FRAM(4A, Ã/16) ≡ FRAM(A, Ã) bit-for-bit for binary graphs (power-of-2 scalings, [M13]).
    inst = config_c1(seed=2)
    r1 = oracle.fram(inst.A, inst.B, None, theta=10.0)
    r2 = oracle.fram(4 * inst.A, inst.B / 16, None, theta=10.0)
    assert r1["passes"] == r2["passes"]
    assert np.array_equal(r1["N"], r2["N"]) and np.array_equal(r1["perm"], r2["perm"])
    r3 = oracle.fram(3 * inst.A, inst.B, None, theta=10.0)
    assert r3["passes"] == r1["passes"] and np.array_equal(r3["perm"], r1["perm"])
    assert np.max(np.abs(r3["N"] - r1["N"])) <= 1e-14


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_exact_recovery_noise_free(seed):
    # Noise-free isomorphic pair (BASELINE acceptance): Φ(M) = Φ(M*), and the planted
    # permutation itself when A has no automorphism-creating structure (R19).
    rng = np.random.Generator(np.random.PCG64(100 + seed))
    n = 40
    A = ba_graph(rng, n, 3)
    sigma = rng.permutation(n)
    B = np.empty_like(A)
    B[np.ix_(sigma, sigma)] = A
    out = oracle.fram(A, B, None, theta=10.0)
    phi = oracle.objective_perm(A, B, None, out["perm"])
    phi_true = oracle.objective_perm(A, B, None, sigma)
    assert phi == phi_true
    assert out["converged"]
    assert np.all(out["N"] >= 0)


@pytest.mark.parametrize("seed", range(4))
def test_brute_force_qap_small(seed):
    # n ≤ 8: Φ(M_FRAM) ≤ Φ_opt always; equal on planted noise-free instances.
    rng = np.random.Generator(np.random.PCG64(seed))
    n = 7
    A = _sym(rng, n, 0.6)
    sigma = rng.permutation(n)
    B = np.empty_like(A)
    B[np.ix_(sigma, sigma)] = A
    out = oracle.fram(A, B, None, theta=10.0)
    _, best = qap_brute_force(A, B)
    phi = oracle.objective_perm(A, B, None, out["perm"])
    assert phi <= best + 1e-12
    assert abs(phi - best) <= 1e-12


def test_fram_invariants_and_determinism(rng):
    inst = config_c1(seed=0)
    r1 = oracle.fram(inst.A, inst.B, None, theta=10.0)
    r2 = oracle.fram(inst.A, inst.B, None, theta=10.0)
    assert np.array_equal(r1["N"], r2["N"]) and r1["passes"] == r2["passes"]
    assert np.all(r1["N"] >= 0)
    n = inst.n
    # |ΣN/n − 1| ≤ γ_th when no SDSN call was capped
    assert max(r1["passes"]) < 1000
    assert abs(r1["N"].sum() / n - 1) <= 1e-3


def test_replay_reproduces(rng):
    inst = config_c1(seed=1)
    r1 = oracle.fram(inst.A, inst.B, None, theta=10.0, keep_trace=True)
    r2 = oracle.fram(inst.A, inst.B, None, theta=10.0, replay=r1["passes"], keep_trace=True)
    assert np.array_equal(r1["N"], r2["N"]) and r2["outer_iters"] == r1["outer_iters"]


# ---------------------------------------------------------------- attributed / unequal sizes (R30)
def test_unary_from_features_definition(rng):
    # K = F F̃ᵀ written out as the feature-term inner product of Eq.(1): ⟨NᵀF, F̃⟩ = ⟨N, K⟩
    F = rng.random((5, 3))
    Ft = rng.random((7, 3))
    K = oracle.unary_from_features(F, Ft)
    for i in range(5):
        for j in range(7):
            assert abs(K[i, j] - sum(F[i, k] * Ft[j, k] for k in range(3))) <= 1e-15
    N = rng.random((5, 7))
    assert abs(np.sum((N.T @ F) * Ft) - np.sum(N * K)) <= 1e-12


def test_padding_is_inert_for_the_real_nodes(rng):
    # Isolated zero-attribute padding nodes add nothing to Φ: for any matching of the padded problem,
    # Φ_padded(M) equals Φ of the original graphs restricted to the real-to-real pairs.
    n1, n2, m, d = 6, 8, 8, 4
    A = rng.random((n1, n1)); A = A + A.T
    B = rng.random((n2, n2)); B = B + B.T
    F, Ft = rng.random((n1, d)), rng.random((n2, d))
    Ap, Bp, Kp = oracle.pad_attributed(A, B, F, Ft, m)
    assert np.all(Ap[n1:] == 0) and np.all(Ap[:, n1:] == 0) and np.all(Kp[n1:] == 0)
    perm = rng.permutation(m)
    real = perm[:n1] < n2
    K = oracle.unary_from_features(F, Ft)
    pr = perm[:n1]
    phi = 0.5 * sum(A[i, j] * B[pr[i], pr[j]] for i in range(n1) for j in range(n1) if real[i] and real[j]) + \
        sum(K[i, pr[i]] for i in range(n1) if real[i])
    assert abs(oracle.objective_perm(Ap, Bp, Kp, perm) - phi) <= 1e-12


def test_fram_attributed_recovers_planted_subgraph():
    # G is an induced subgraph of G̃ (n1 < n2) with matching nonnegative features (K = FF̃ᵀ ≥ 0, as
    # the method requires): FRAM on the padded problem recovers the planted embedding (R30).
    rng = np.random.Generator(np.random.PCG64(77))
    n2, n1, d = 30, 24, 8
    B = (rng.random((n2, n2)) < 0.25).astype(float)
    B = np.triu(B, 1); B = B + B.T
    Ft = np.maximum(0.0, rng.normal(size=(n2, d)))
    emb = rng.permutation(n2)[:n1]
    A = B[np.ix_(emb, emb)]
    F = Ft[emb]
    out = oracle.fram_attributed(A, B, F, Ft, n2, lam=1.0, theta=10.0)
    assert np.array_equal(out["perm_attr"], emb)


def test_matching_error_hand_computed():
    # ½‖A − MÃMᵀ‖_F + ‖F − MF̃‖_F, (MÃMᵀ)_ij = Ã[perm i, perm j], (MF̃)_i = F̃[perm i].
    A = np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], float)      # path 0-1-2
    B = np.array([[0, 1, 1], [1, 0, 0], [1, 0, 0]], float)      # star centred at 0
    F = np.array([[1.0], [2.0], [3.0]])
    Ft = np.array([[2.0], [1.0], [5.0]])
    # identity: A − B has four unit entries → ½·2 = 1; F − F̃ = (−1, 1, −2) → √6
    assert oracle.matching_error(A, B, [0, 1, 2]) == 1.0
    assert abs(oracle.matching_error(A, B, [0, 1, 2], F, Ft) - (1.0 + np.sqrt(6.0))) <= 1e-15
    # perm (1, 0, 2) maps the path's centre onto the star's centre: MÃMᵀ = A; F̃[perm] = (1, 2, 5)
    assert oracle.matching_error(A, B, [1, 0, 2]) == 0.0
    assert oracle.matching_error(A, B, [1, 0, 2], F, Ft) == 2.0
