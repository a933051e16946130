"""LAP discretisation oracle, FP64 — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq.(2): M = argmin_{P∈Π} ‖P − N‖_F  ⇔  argmax_P ⟨P, N⟩ because ‖P‖²_F = n on Π
(S:312).  Alg.1 step 10 and §6 "Complexity" name the Hungarian method
(Kuhn 1955).  R17 fixes *which* Hungarian: shortest-augmenting-path Kuhn–Munkres with row
and column potentials on C = −N, rows inserted in order, ties to the lowest column index.
The GPU kernel K7 must reproduce these choices bit-for-bit (every float op is an FP64 add or
subtract in the same association order).

Pins: brute_force_max at n ≤ 8 (score always; permutation when the optimum is unique);
scipy.optimize.linear_sum_assignment score equality (an independent library LAP);
permutation-matrix round trip; SPEC examples S:282-304.
"""
from __future__ import annotations

import itertools

import numpy as np


def perm_score(N, perm):
    """Σ_i N[i, perm[i]] summed in row order."""
    N = np.asarray(N, np.float64)
    s = 0.0
    for i, j in enumerate(perm):
        s += float(N[i, j])
    return s


def lap_max(N):
    """perm = argmax_π Σ_i N[i, π(i)] by the R17 Hungarian (SURVEY §8(c) "LAP_max, exactly").

    1-based potentials u[0..n], v[0..n]; p[j] = row owning column j (0 = free); column 0 virtual.
    for i = 1..n: p[0]=i; j0=0; minv=+inf; used=false
      repeat: used[j0]=true; i0=p[j0]; delta=+inf
              for j=1..n, !used[j]: cur=(C[i0][j]−u[i0])−v[j]; if cur<minv[j]: minv[j]=cur, way[j]=j0
                                     if minv[j]<delta: delta=minv[j], j1=j      (strict ⇒ lowest j)
              for j=0..n: used ? (u[p[j]]+=delta, v[j]−=delta) : minv[j]−=delta
              j0=j1
      until p[j0]==0;  augment along way[].
    The inner j-loop is evaluated elementwise over j (each j's update is independent; the
    sequential first-minimum equals numpy's first argmin) — same arithmetic, same order per j.
    Returns perm (int64, 0-based): perm[i] = column matched to row i.
    """
    N = np.asarray(N, dtype=np.float64)
    n = N.shape[0]
    if N.ndim != 2 or N.shape[1] != n:
        raise ValueError("N must be square")
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    C = -N
    INF = np.inf
    u = np.zeros(n + 1)
    v = np.zeros(n + 1)
    p = np.zeros(n + 1, dtype=np.int64)
    way = np.zeros(n + 1, dtype=np.int64)
    for i in range(1, n + 1):
        p[0] = i
        j0 = 0
        minv = np.full(n + 1, INF)
        used = np.zeros(n + 1, dtype=bool)
        while True:
            used[j0] = True
            i0 = p[j0]
            free = ~used[1:]
            cur = (C[i0 - 1, :] - u[i0]) - v[1:]
            upd = free & (cur < minv[1:])
            minv[1:][upd] = cur[upd]
            way[1:][upd] = j0
            masked = np.where(free, minv[1:], INF)
            j1 = int(np.argmin(masked)) + 1
            delta = masked[j1 - 1]
            uj = np.nonzero(used)[0]
            u[p[uj]] += delta
            v[uj] -= delta
            minv[~used] -= delta
            j0 = j1
            if p[j0] == 0:
                break
        while True:
            j1 = way[j0]
            p[j0] = p[j1]
            j0 = j1
            if j0 == 0:
                break
    perm = np.empty(n, dtype=np.int64)
    for j in range(1, n + 1):
        perm[p[j] - 1] = j - 1
    return perm


def brute_force_max(N):
    """Exhaustive argmax over all n! permutations (n ≤ 8); ties → lexicographically smallest perm
    (S:286-294).  Returns (perm, score)."""
    N = np.asarray(N, np.float64)
    n = N.shape[0]
    if n > 8:
        raise ValueError("brute force limited to n <= 8")
    best, best_s = None, -np.inf
    for perm in itertools.permutations(range(n)):
        s = perm_score(N, perm)
        if s > best_s:
            best, best_s = perm, s
    return np.array(best, dtype=np.int64), best_s
