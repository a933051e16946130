"""Exact references used only to pin the oracle — TEST INFRASTRUCTURE ONLY.

* dykstra_project: the exact Euclidean projection P_D(X) onto the Birkhoff polytope
  (Eq.(4)) by Dykstra's alternating projection with corrections.
  SDSN does NOT compute this (R8, [M9]); it pins Theorems 1 and 3 only.
* affine_projection_kkt: the equality-constrained least-squares problem behind P1
  (proof P:793-859) solved as a KKT linear system.
* qap_brute_force: max Φ(M) over all permutations (Eq.(1)), n ≤ 8.
"""
from __future__ import annotations

import itertools

import numpy as np


def dykstra_project(Y, tol=1e-13, max_iters=200000):
    """P_D(Y) by Dykstra: Z = P1(X+p); p = X+p−Z; X' = max(0, Z+q); q = Z+q−X'.

    Uses its own P1 (row/column-sum closed form) so it shares nothing with fram_oracle.
    Returns (D, converged)."""
    Y = np.asarray(Y, np.float64)
    n = Y.shape[0]

    def p1(X):
        r = X.sum(axis=1, keepdims=True)
        c = X.sum(axis=0, keepdims=True)
        return X + 1.0 / n + X.sum() / n**2 - r / n - c / n

    X = Y.copy()
    p = np.zeros_like(Y)
    q = np.zeros_like(Y)
    for _ in range(max_iters):
        Z = p1(X + p)
        p = X + p - Z
        Xn = np.maximum(0.0, Z + q)
        q = Z + q - Xn
        if np.max(np.abs(Xn - X)) < tol:
            return Xn, True
        X = Xn
    return X, False


def affine_projection_kkt(X):
    """argmin_Y ‖Y − X‖_F s.t. Y1 = 1, Yᵀ1 = 1, solved as the KKT system.

    Constraint matrix C (2n × n²) acting on vec(Y) (row-major); Y = X − Cᵀλ with
    (C Cᵀ) λ = C vec(X) − 1, solved by least squares (C Cᵀ has rank 2n−1)."""
    X = np.asarray(X, np.float64)
    n = X.shape[0]
    C = np.zeros((2 * n, n * n))
    for i in range(n):
        C[i, i * n:(i + 1) * n] = 1.0          # row sums
        C[n + i, i::n] = 1.0                   # column sums
    x = X.reshape(-1)
    rhs = C @ x - np.ones(2 * n)
    lam, *_ = np.linalg.lstsq(C @ C.T, rhs, rcond=None)
    return (x - C.T @ lam).reshape(n, n)


def qap_brute_force(A, B, K=None, lam=1.0):
    """max over permutations of Φ(M) = ½Σ A_ij Ã_{πi,πj} + λΣ K_{i,πi}  (n ≤ 8).  Returns (perm, Φ)."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    n = A.shape[0]
    if n > 8:
        raise ValueError("n <= 8")
    best, best_v = None, -np.inf
    for perm in itertools.permutations(range(n)):
        P = np.array(perm)
        v = 0.5 * float(np.sum(A * B[np.ix_(P, P)]))
        if K is not None:
            v += lam * float(np.sum(np.asarray(K)[np.arange(n), P]))
        if v > best_v + 1e-12:
            best, best_v = P, v
    return best, best_v
