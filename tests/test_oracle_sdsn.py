"""Pins for the oracle's SDSN (Alg. 2) — closed forms, invariants, theorems."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.exact import dykstra_project
from oracle.lap import brute_force_max, lap_max
from synth import random_nonneg, random_perm_matrix

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _closed_form_cases():
    with open(os.path.join(GOLD, "sdsn_closed_form_A.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _closed_form_cases(), ids=lambda c: f"n{c['n']}")
def test_closed_form_A_identity(case):
    n, th, g = case["n"], case["theta"], case["gamma_th"]
    D, k = oracle.sdsn(np.eye(n), th, gamma_th=g, sdsn_max=100000)
    assert k == case["passes"]
    # independent closed form d_k = 1 + (θ/2−1)(1−1/n)^k
    d = 1.0 + (th / 2 - 1) * (1 - 1.0 / n) ** k
    assert np.all(np.abs(np.diag(D) - d) <= 1e-14)
    if case["diag"] is not None:
        assert abs(D[0, 0] - case["diag"]) <= 2e-15
    off = D - np.diag(np.diag(D))
    assert np.all(off == 0.0)
    kstar = max(1, math.ceil(math.log(g / (th / 2 - 1)) / math.log(1 - 1.0 / n)))
    assert k == kstar + 1


@pytest.mark.parametrize("n", [4, 8, 16, 64, 5, 7, 100])
def test_closed_form_B_permutation_fixed_point(rng, n):
    # SDSN(P, θ=2) = P in 2 passes; bit-exact for n = 2^k, ≤ 1 ulp otherwise ([M15]).
    P = random_perm_matrix(rng, n)
    D, k = oracle.sdsn(P, 2.0)
    assert k == 2
    tol = 0.0 if (n & (n - 1)) == 0 else 2.3e-16
    assert np.max(np.abs(D - P)) <= tol


def test_zero_input_returns_uniform():
    D, k = oracle.sdsn(np.zeros((5, 5)), 10.0)
    assert k == 0 and np.all(D == 0.2)


def test_negative_input_rejected():
    with pytest.raises(oracle.DataError):
        oracle.sdsn(-np.eye(3), 2.0)


@pytest.mark.parametrize("kind", ["uniform", "sparse", "lowrank", "spiky"])
def test_per_pass_invariants(rng, kind):
    # After every pass: Y ≥ 0; all row/col sums ≥ 1 − O(u); Σ(r−1) = Σ(c−1) = n·γ_next
    # (mass identity, App. B.1); γ nonincreasing for j ≥ 1 ([M9]).
    n, th = 12, 10.0
    X = random_nonneg(rng, n, kind)
    _, kmax, gams = oracle.sdsn(X, th, gamma_th=1e-6, sdsn_max=400, return_gammas=True)
    for j in range(1, min(kmax, 60) + 1):
        Y, _ = oracle.sdsn(X, th, sdsn_fixed=j)
        assert np.all(Y >= 0)
        r, c = Y.sum(1), Y.sum(0)
        assert r.min() >= 1 - 1e-12 and c.min() >= 1 - 1e-12
        mass = Y.sum() - n
        assert abs((r - 1).sum() - mass) <= 1e-12 and abs((c - 1).sum() - mass) <= 1e-12
        if j < len(gams):
            assert abs(gams[j] - (Y.sum() / n - 1)) <= 1e-13
    g = np.array(gams[1:])
    assert np.all(np.diff(g) <= 1e-14)


def test_theorem4_small_theta(rng):
    # Thm 4 (proof P:778-790): θ → 0 ⇒ D → 11ᵀ/n.
    for n in (5, 10, 20):
        X = rng.random((n, n))
        D, _ = oracle.sdsn(X, 1e-6, gamma_th=1e-12, sdsn_max=10000)
        assert np.linalg.norm(D - 1.0 / n) <= 1e-5


def test_theorem2_gap_bound(rng):
    # Thm 2 (R25): ε = (⟨D∞, X̂⟩ − ⟨Dθ, X̂⟩)/n ≤ 1/θ with X̂ = X/max X, D∞ a LAP optimum.
    for trial in range(30):
        n = int(rng.integers(3, 9))
        X = rng.random((n, n))
        Xh = X / X.max()
        perm, best = brute_force_max(Xh)
        for th in (1.0, 2.0, 10.0):
            D, _ = oracle.sdsn(X, th, gamma_th=1e-10, sdsn_max=200000)
            eps = (best - float(np.sum(D * Xh))) / n
            assert eps <= 1.0 / th + 1e-9


def test_scale_invariance(rng):
    # P:116-142 motivation; SDSN(wX) = SDSN(X): bit-exact for w = 2^k ([M13]).
    X = rng.random((9, 9))
    D1, k1 = oracle.sdsn(X, 10.0)
    D2, k2 = oracle.sdsn(16.0 * X, 10.0)
    assert k1 == k2 and np.array_equal(D1, D2)
    D3, k3 = oracle.sdsn(3.7 * X, 10.0)
    assert k3 == k1 and np.max(np.abs(D3 - D1)) <= 1e-14


def test_permutation_equivariance(rng):
    n = 10
    X = rng.random((n, n))
    P = random_perm_matrix(rng, n)
    Q = random_perm_matrix(rng, n)
    D, _ = oracle.sdsn(X, 10.0, sdsn_fixed=50)
    Dp, _ = oracle.sdsn(P @ X @ Q, 10.0, sdsn_fixed=50)
    assert np.max(np.abs(Dp - P @ D @ Q)) <= 1e-14


def test_passes_grow_with_theta(rng):
    # Iteration-count theorem: passes grow with θ ([M1]).
    X = rng.random((40, 40))
    ks = [oracle.sdsn(X, th, gamma_th=1e-6, sdsn_max=100000)[1] for th in (2.0, 10.0, 50.0)]
    assert ks[0] < ks[1] < ks[2]


def test_sdsn_is_not_the_exact_projection(rng):
    # R8: SDSN's limit differs from the Dykstra projection (measured gap [M9]); Dykstra satisfies
    # KKT: D = max(0, Y − u1ᵀ − 1vᵀ) and is DS.
    n = 6
    X = rng.random((n, n))
    Y = 5.0 * X / X.max()
    Dd, ok = dykstra_project(Y)
    assert ok
    assert np.max(np.abs(Dd.sum(0) - 1)) <= 1e-12 and np.max(np.abs(Dd.sum(1) - 1)) <= 1e-12
    Ds, _ = oracle.sdsn(X, 10.0, gamma_th=1e-13, sdsn_max=10 ** 6)
    assert np.linalg.norm(Ds - Dd) > 1e-6


def test_dykstra_reference():
    D, ok = dykstra_project(np.diag([2.0, 2.0]))
    assert ok and np.max(np.abs(D - np.eye(2))) <= 1e-12


def test_dsn_fixed(rng):
    U = np.full((6, 6), 1 / 6)
    assert np.max(np.abs(oracle.dsn_fixed(U, 7) - U)) <= 1e-15
    assert np.max(np.abs(oracle.dsn_fixed(np.zeros((4, 4)), 1) - 0.25)) <= 1e-15
    X = rng.random((8, 8))
    assert oracle.gamma(oracle.dsn_fixed(X, 200)) <= oracle.gamma(oracle.dsn_fixed(X, 30)) + 1e-15


def test_lap_recovers_planted_from_sdsn(rng):
    # θ large, near-permutation input: the LAP of the SDSN output is the planted permutation.
    n = 30
    P = random_perm_matrix(rng, n)
    X = P * 3 + rng.random((n, n))
    D, _ = oracle.sdsn(X, 10.0)
    assert np.array_equal(lap_max(D), np.argmax(P, axis=1))


# ---- FP32-stored SDSN (the emulated-rounding diagnostic reference) ----
@pytest.mark.parametrize("n", [4, 8, 64, 256])
def test_sdsn_fp32_closed_form_B_bitexact(rng, n):
    # SDSN(P, θ=2) = P: every quantity (1/n, S/n², a, b) is a power of two for n = 2^k, so exact in FP32
    P = random_perm_matrix(rng, n)
    D, k = oracle.sdsn_fp32(P, 2.0)
    assert k == 2 and np.array_equal(D, P)


@pytest.mark.parametrize("n", [4, 32, 1024])
def test_sdsn_fp32_uniform_input(n):
    # X = c·11ᵀ: Y⁰ = θ/2 everywhere, a = 1/n, b = −θ/2, so Y¹ = 11ᵀ/n exactly (n = 2^k); γ₁ = 0 stops
    # after pass 2 (R5) with 11ᵀ/n unchanged.
    D, k, g = oracle.sdsn_fp32(np.full((n, n), 3.0), 10.0, return_gammas=True)
    assert k == 2 and np.all(D == 1.0 / n) and g[1] == 0.0


def test_sdsn_fp32_is_fp32_and_close_to_fp64(rng):
    # storage is FP32 (every output value round-trips through float32), and the deviation from the FP64
    # oracle after k passes stays within the FP32 rounding bound: each pass adds ≤ 2 roundings of
    # relative size u32 to |Y| ≤ θ/2 and the pass map is nonexpansive ([M22]) ⇒ ≤ 2·k·u32·θ/2.
    n, th, k = 50, 10.0, 60
    X = random_nonneg(rng, n, "uniform").astype(np.float32).astype(np.float64)
    D32, k32 = oracle.sdsn_fp32(X, th, sdsn_fixed=k)
    D64, _ = oracle.sdsn(X, th, sdsn_fixed=k)
    assert k32 == k
    assert np.array_equal(D32, D32.astype(np.float32).astype(np.float64))
    err = np.max(np.abs(D32 - D64))
    assert 0 < err <= 2 * k * 2.0 ** -24 * th / 2
    assert np.all(D32 >= 0)


def test_dsn_fixed_one_round_is_p2_of_p1(rng):
    # DSPFP's DSN has no θ-scaling: one round is P2(P1(X)) of the raw X.  A non-uniform X
    # with entries far from 1/n distinguishes it from the θ-scaled SDSN.
    n = 9
    X = rng.random((n, n)) * 7.0
    X[2, 3] = 40.0
    one = oracle.p2_nonneg(oracle.p1_project(X))
    assert np.allclose(oracle.dsn_fixed(X, 1), one, rtol=0, atol=1e-13)
    assert np.allclose(oracle.dsn_fixed(X, 2), oracle.p2_nonneg(oracle.p1_project(one)), rtol=0, atol=1e-13)
    Ds, _ = oracle.sdsn(X, 2.0, sdsn_fixed=1)
    assert np.max(np.abs(Ds - one)) > 1e-3           # θ-scaled SDSN differs: the scaling is really skipped
