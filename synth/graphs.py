"""Seeded synthetic graph-matching instances (BASELINE.json configs C1-C5).

All randomness comes from numpy.random.Generator(PCG64(seed)), drawn in the fixed order
graph → noise → σ → features.  Ground truth orientation (R18): B[σ(i), σ(j)] = A_noisy[i, j],
so the planted matching is perm_true[i] = σ(i) (M[i, σ(i)] = 1).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Schedules of SURVEY.md §8(d) (R3, R4): θ per config, α=0.95, λ=1.
SCHEDULES = {
    "default": dict(alpha=0.95, gamma_th=1e-3, delta_th=1e-4, max_outer=100, sdsn_max=1000),
    "uncapped": dict(alpha=0.95, gamma_th=1e-3, delta_th=1e-4, max_outer=100, sdsn_max=20000),
    "loose": dict(alpha=0.95, gamma_th=1e-1, delta_th=1e-4, max_outer=100, sdsn_max=1000),
}


@dataclass
class Instance:
    name: str
    A: np.ndarray                 # n×n, symmetric, ≥0 (float64, or float32 holding bf16 values for C5)
    B: np.ndarray                 # Ã = P·A_noisy·Pᵀ
    K: np.ndarray | None          # unary term (None ⇒ 0)
    perm_true: np.ndarray         # σ, int64
    theta: float
    lam: float = 1.0
    inlier_mask: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.A.shape[0]


def _permute(Anoisy, sigma):
    n = Anoisy.shape[0]
    B = np.empty_like(Anoisy)
    B[np.ix_(sigma, sigma)] = Anoisy          # B[σ(i), σ(j)] = A_noisy[i, j]
    assert B.shape == (n, n)
    return B


def er_graph(rng, n, p, weighted=False):
    """Erdős–Rényi: each upper-triangle pair is an edge independently with prob. p; symmetric,
    zero diagonal; weights U(0,1) if weighted (drawn after the mask)."""
    iu = np.triu_indices(n, 1)
    mask = rng.random(len(iu[0])) < p
    w = rng.random(int(mask.sum())) if weighted else np.ones(int(mask.sum()))
    A = np.zeros((n, n))
    A[iu[0][mask], iu[1][mask]] = w
    return A + A.T


def ba_graph(rng, n, m=5):
    """Barabási–Albert, m edges per new node: nodes 0..m−1 start isolated; node m attaches to
    0..m−1; later nodes draw targets uniformly from the multiset of edge endpoints, re-drawing
    duplicates.  |E| = m(n−m).  Returns a binary symmetric dense matrix."""
    A = np.zeros((n, n))
    endpoints = []
    for v in range(m, n):
        if v == m:
            targets = list(range(m))
        else:
            targets = []
            seen = set()
            while len(targets) < m:
                t = endpoints[int(rng.integers(len(endpoints)))]
                if t not in seen:
                    seen.add(t)
                    targets.append(t)
        for t in targets:
            A[v, t] = A[t, v] = 1.0
            endpoints.append(v)
            endpoints.append(t)
    return A


def _rewire(rng, A, frac, new_weight=None):
    """Remove k = round(frac·|E|) uniformly chosen edges and add k uniformly chosen non-edges of
    the original graph (edge count preserved).  Added edges get weight 1 or new_weight(rng)."""
    n = A.shape[0]
    iu, ju = np.nonzero(np.triu(A, 1))
    E = len(iu)
    k = int(round(frac * E))
    rem = rng.choice(E, size=k, replace=False)
    An = A.copy()
    An[iu[rem], ju[rem]] = 0.0
    An[ju[rem], iu[rem]] = 0.0
    added = set()
    while len(added) < k:
        i, j = (int(x) for x in rng.integers(0, n, size=2))
        if i == j:
            continue
        if i > j:
            i, j = j, i
        if A[i, j] != 0.0 or (i, j) in added:
            continue
        added.add((i, j))
        w = 1.0 if new_weight is None else new_weight(rng)
        An[i, j] = An[j, i] = w
    return An


def config_c1(seed=0):
    """C1: n=20 binary ER(p=0.2); 'flip 5% of edges symmetrically' = toggle round(0.05|E|)
    unordered pairs drawn without replacement from all n(n−1)/2 pairs; K = 0; θ = 10 (R4)."""
    n = 20
    rng = np.random.Generator(np.random.PCG64(seed))
    A = er_graph(rng, n, 0.2)
    E = int(np.triu(A, 1).sum())
    iu = np.triu_indices(n, 1)
    k = int(round(0.05 * E))
    tog = rng.choice(len(iu[0]), size=k, replace=False)
    An = A.copy()
    for t in tog:
        i, j = iu[0][t], iu[1][t]
        An[i, j] = An[j, i] = 1.0 - An[i, j]
    sigma = rng.permutation(n)
    return Instance("C1", A, _permute(An, sigma), None, sigma.astype(np.int64), theta=10.0)


def config_c2(seed=0, n=500):
    """C2: weighted ER(p=0.05), w~U(0,1); Ã: |w + N(0,0.05²)| on existing edges, then delete
    round(0.1|E|) uniformly chosen edges; K = 0; θ = 10."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A = er_graph(rng, n, 0.05, weighted=True)
    iu, ju = np.nonzero(np.triu(A, 1))
    An = A.copy()
    w = np.abs(A[iu, ju] + rng.normal(0.0, 0.05, size=len(iu)))
    An[iu, ju] = w
    An[ju, iu] = w
    k = int(round(0.1 * len(iu)))
    rem = rng.choice(len(iu), size=k, replace=False)
    An[iu[rem], ju[rem]] = 0.0
    An[ju[rem], iu[rem]] = 0.0
    sigma = rng.permutation(n)
    return Instance("C2", A, _permute(An, sigma), None, sigma.astype(np.int64), theta=10.0)


def config_c3_instance(seed_seq, n=64, d=32):
    """C3 instance: points p~U[0,1]²; A_ij = exp(−‖p_i−p_j‖²/0.05); graph 2: q_{σ(i)} = p_i +
    N(0, 0.02² I) (R27: 0.02 is the std); 10% outliers: round(0.1n) graph-2 slots replaced by
    fresh U[0,1]² points and fresh features; f_i ~ N(0, I/d); g_{σ(i)} = f_i + N(0, 0.1² I/d);
    K_ij = exp(−‖f_i − g_j‖²); θ = 2 (dense, R4).  Accuracy over inlier rows (R20)."""
    rng = np.random.Generator(np.random.PCG64(seed_seq))
    P = rng.random((n, 2))
    Q0 = P + rng.normal(0.0, 0.02, size=(n, 2))
    sigma = rng.permutation(n)
    n_out = int(round(0.1 * n))
    out_slots = rng.choice(n, size=n_out, replace=False)
    Q = np.empty_like(Q0)
    Q[sigma] = Q0
    Q[out_slots] = rng.random((n_out, 2))
    F = rng.normal(0.0, 1.0 / np.sqrt(d), size=(n, d))
    G0 = F + rng.normal(0.0, 0.1 / np.sqrt(d), size=(n, d))
    Gf = np.empty_like(G0)
    Gf[sigma] = G0
    Gf[out_slots] = rng.normal(0.0, 1.0 / np.sqrt(d), size=(n_out, d))

    def kern(X, Y, h):
        D2 = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
        return np.exp(-D2 / h)

    A = kern(P, P, 0.05)
    B = kern(Q, Q, 0.05)
    K = kern(F, Gf, 1.0)
    inv = np.empty(n, dtype=np.int64)
    inv[sigma] = np.arange(n)
    inlier = np.ones(n, dtype=bool)
    inlier[inv[out_slots]] = False          # rows i whose partner slot σ(i) was replaced
    return Instance("C3", A, B, K, sigma.astype(np.int64), theta=2.0, inlier_mask=inlier)


def config_c3_batch(batch=4096, n=64, start=0):
    """C3 batch: instance b uses SeedSequence(3).spawn(batch_total)[b]."""
    seqs = np.random.SeedSequence(3).spawn(start + batch)[start:]
    return [config_c3_instance(s, n) for s in seqs]


def config_c4(seed=0, n=4096):
    """C4: Barabási–Albert m=5 (binary, dense storage); Ã with 5% edge rewiring; K = 0; θ = 10."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A = ba_graph(rng, n, 5)
    An = _rewire(rng, A, 0.05)
    sigma = rng.permutation(n)
    return Instance("C4", A, _permute(An, sigma), None, sigma.astype(np.int64), theta=10.0)


def config_ubc(seed=0, n=2000, d=128, jitter=0.01, feat_noise=0.05):
    """NEXT-2 stand-in for the paper's ubc(2000) task (Fig. 3; graphs from images App. F,
    P:1047): FULLY CONNECTED keypoint graphs whose edge attribute is the inter-node Euclidean distance,
    with SIFT-like node attributes.  The UBC images are not available; synthetic recipe:
      points p_i ~ U[0,1]²; graph 2: q_{σ(i)} = R_φ p_i + τ + N(0, jitter² I) with a random rotation φ and
      translation τ (a rigid motion keeps the distances); A_ij = ‖p_i − p_j‖, Ã_kl = ‖q_k − q_l‖;
      features f_i = |z_i|/‖z_i‖, z_i ~ N(0, I_d) (non-negative, unit length like SIFT descriptors);
      f̃_{σ(i)} = |f_i + N(0, feat_noise² I)| renormalised; K = F F̃ᵀ ≥ 0.
    θ = 2 (dense graphs), λ = 1.  Returns an Instance with K = None and F, F̃ in meta."""
    rng = np.random.Generator(np.random.PCG64(seed))
    P = rng.random((n, 2))
    phi = rng.uniform(0.0, 2.0 * np.pi)
    Rm = np.array([[np.cos(phi), -np.sin(phi)], [np.sin(phi), np.cos(phi)]])
    tau = rng.random(2)
    Q0 = P @ Rm.T + tau + rng.normal(0.0, jitter, size=(n, 2))
    sigma = rng.permutation(n)
    Q = np.empty_like(Q0)
    Q[sigma] = Q0
    Z = np.abs(rng.normal(size=(n, d)))
    F = Z / np.linalg.norm(Z, axis=1, keepdims=True)
    G0 = np.abs(F + rng.normal(0.0, feat_noise, size=(n, d)))
    G0 /= np.linalg.norm(G0, axis=1, keepdims=True)
    Ft = np.empty_like(G0)
    Ft[sigma] = G0

    def dist(X):
        D2 = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
        return np.sqrt(np.maximum(D2, 0.0))

    A = dist(P)
    B = dist(Q)
    return Instance("UBC", A, B, None, sigma.astype(np.int64), theta=2.0, meta={"F": F, "Ft": Ft})


def _bf16_values(x):
    import torch
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).to(torch.float32).numpy()


def config_c5(seed=0, n=16384, p=0.01):
    """C5: weighted ER(p=0.01), w~U(0,1) rounded to BF16 (the instance *is* the BF16 values),
    stored dense float32; Ã with 5% rewiring, added edges with fresh BF16-rounded U(0,1)
    weights; K = 0; θ = 10.  Built row by row (Binomial count + positions) to bound memory."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A = np.zeros((n, n), dtype=np.float32)
    for i in range(n - 1):
        m = n - 1 - i
        cnt = rng.binomial(m, p)
        if cnt:
            cols = i + 1 + rng.choice(m, size=cnt, replace=False)
            w = _bf16_values(rng.random(cnt))
            w[w == 0] = np.float32(2.0 ** -8)
            A[i, cols] = w
            A[cols, i] = w
    An = _rewire(rng, A, 0.05, new_weight=lambda r: max(float(_bf16_values(r.random())), 2.0 ** -8))
    sigma = rng.permutation(n)
    return Instance("C5", A, _permute(An.astype(np.float32), sigma), None, sigma.astype(np.int64),
                    theta=10.0)


def random_nonneg(rng, n, kind="uniform"):
    """Generic SDSN test inputs: 'uniform' U[0,1]; 'sparse' (10% nonzero); 'lowrank' rank-1
    degree-like (the first FRAM gradient d·d̃ᵀ/n); 'spiky' near-permutation + noise."""
    if kind == "uniform":
        return rng.random((n, n))
    if kind == "sparse":
        return rng.random((n, n)) * (rng.random((n, n)) < 0.1)
    if kind == "lowrank":
        return np.outer(rng.random(n) + 0.1, rng.random(n) + 0.1)
    if kind == "spiky":
        P = random_perm_matrix(rng, n)
        return P * 5.0 + rng.random((n, n)) * 0.5
    raise ValueError(kind)


def random_perm_matrix(rng, n):
    P = np.zeros((n, n))
    P[np.arange(n), rng.permutation(n)] = 1.0
    return P
