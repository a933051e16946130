"""FRAM / SDSN oracle, FP64, NumPy — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows Algorithm 1 (FRAM) and Algorithm 2 (SDSN) step
by step in the paper's order and notation, with the readings R1-R29 of
DESIGN.md §3 where the paper is silent or garbled.  Everything is FP64 and
unfused: a library primitive (matmul, sum, maximum) may serve as one step, but
no blocking, fusion or reordering beyond what the algorithm states.

Pins (tests/test_oracle_*.py, all `-m "not gpu"`):
  precondition  — identity (A'NÃ'+λK') = (ANÃ+λK)/c; c=1 leaves inputs unchanged.
  gradient      — triple-loop definition at n<=12; A'=Ã'=I => G = N + λK'.
  p1_project    — KKT equality-constrained least squares (exact.affine_projection_kkt),
                  P1(0)=11ᵀ/n, idempotence, P1−P3 = 11ᵀ/n (Lemma).
  p2_nonneg     — definition examples.
  sdsn          — closed form A (SDSN(I_n), golden file), closed form B
                  (SDSN(P,θ=2)=P), per-pass invariants, Thm 2/Thm 4
                  limits, scale invariance, permutation equivariance.
  fram          — closed form C (A=Ã=0), scale invariance, exact recovery on
                  noise-free isomorphic pairs, brute-force QAP at n<=8.
  sdsn_fp32     — closed form B bit-exact in FP32 (n = 2^k), the uniform-input closed form
                  (11ᵀ/n in 2 passes), FP32 storage, deviation from `sdsn` within the FP32
                  rounding bound (tests/test_oracle_sdsn.py).
  dsn_fixed     — one round = P2(P1(X)) on a non-uniform X (no θ-scaling).
  matching_error— hand-computed 3-node example with and without the feature term.
  objective_perm, node_accuracy — tests/test_oracle_fram.py (brute force, planted recovery).
"""
from __future__ import annotations

import numpy as np


class DataError(ValueError):
    """Invalid input data (non-finite, negative, c = max(A,Ã,K) = 0): S:99-100."""


def _check_square(X, name="X"):
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] != X.shape[1]:
        raise ValueError(f"{name} must be square, got {X.shape}")
    return X


# --------------------------------------------------------------------------------------
# Alg. 1 steps 2-3: preconditioning (rationale P:1025)
# --------------------------------------------------------------------------------------
def precondition(A, B, K=None):
    """c = max(A, Ã, K); A' = A/√c, Ã' = Ã/√c, K' = K/c  — all FP64 (Alg.1 steps 2-3).

    R7: applied as written even though c cancels after SDSN's own max-normalisation.
    K=None means K = 0 (no unary term).  Returns (A', Ã', K', c).
    """
    A = _check_square(A, "A")
    B = _check_square(B, "B")
    n = A.shape[0]
    if B.shape != A.shape:
        raise ValueError("A and Ã must have the same shape")
    Kz = np.zeros((n, n)) if K is None else _check_square(K, "K")
    for M, nm in ((A, "A"), (B, "Ã"), (Kz, "K")):
        if not np.all(np.isfinite(M)):
            raise DataError(f"{nm} has non-finite entries")
        if np.any(M < 0):
            raise DataError(f"{nm} has negative entries")
    c = max(float(A.max()), float(B.max()), float(Kz.max()))
    if c == 0.0:
        raise DataError("c = max(A, Ã, K) = 0 (S:344)")
    sA = np.sqrt(c)                      # IEEE division by the rounded sqrt (O2)
    return A / sA, B / sA, Kz / c, c


# --------------------------------------------------------------------------------------
# Alg. 1 step 5: gradient X = A N Ã + λK (Eq.(3))
# --------------------------------------------------------------------------------------
def gradient(Ap, N, Bp, Kp, lam):
    """X⁽ᵗ⁾ = A' N⁽ᵗ⁻¹⁾ Ã' + λK'  (Alg.1 step 5).  Library matmul as one step."""
    G = (Ap @ N) @ Bp
    return G + lam * Kp


# --------------------------------------------------------------------------------------
# §5.1 projections P1, P2 (Eq. P1_sol) and Lemma P3
# --------------------------------------------------------------------------------------
def p1_project(X):
    """P1(X) = X + (I/n + 1ᵀX1/n² I − X/n) 11ᵀ − 11ᵀX/n   (written out as matrices).

    Euclidean projection onto {Y1 = Yᵀ1 = 1}; valid for asymmetric X (Theorem).
    """
    X = _check_square(X)
    n = X.shape[0]
    I = np.eye(n)
    one = np.ones((n, n))
    S = X.sum()
    return X + (I / n + (S / n**2) * I - X / n) @ one - (one @ X) / n


def p3_project(X):
    """P3(X) = X + (1ᵀX1/n² I − X/n) 11ᵀ − 11ᵀX/n   (Lemma): zero-marginal projection."""
    X = _check_square(X)
    n = X.shape[0]
    I = np.eye(n)
    one = np.ones((n, n))
    S = X.sum()
    return X + ((S / n**2) * I - X / n) @ one - (one @ X) / n


def p2_nonneg(X):
    """P2(X) = (X + |X|)/2 = max(0, X)."""
    X = np.asarray(X, dtype=np.float64)
    return (X + np.abs(X)) / 2.0


def gamma(X):
    """γ(X) = 1ᵀX1/n − 1."""
    X = _check_square(X)
    return X.sum() / X.shape[0] - 1.0


# --------------------------------------------------------------------------------------
# Alg. 2 SDSN
# --------------------------------------------------------------------------------------
def sdsn(X, theta, gamma_th=1e-3, sdsn_max=1000, sdsn_fixed=0, scale=True,
         check_nonneg=True, return_gammas=False):
    """SDSN(X, θ) — Algorithm 2, literally, FP64.

    Step 1: X⁽⁰⁾ = (θ/2) X / max(X), evaluated as s = (θ/2)/max X, Y = s·X (R11).
      All-zero X returns 11ᵀ/n with 0 passes (R10).  `scale=False` skips this step
      (DSPFP's plain DSN; NEXT-1).
    Loop (steps 3-7), pass j on input Y_j:
      r = Y1, c = 1ᵀY, S = 1ᵀY1                 (S3; sums in FP64, R13)
      γ_j = S/n − 1                             (step 7, lagged: mass of the pass input)
      a_i = (1/n + S/n²) − r_i/n ; b_j = −c_j/n (steps 3-5 expanded elementwise, R9)
      Y_{j+1} = max(0, (Y_j + a) + b)           (step 6, P2)
    Stop after pass j (0-based) iff (j ≥ 1 and γ_j ≤ γ_th) or j+1 = sdsn_max (R5, R16);
    with sdsn_fixed > 0: exactly sdsn_fixed passes (DSPFP / replay).
    Returns (D, passes[, gammas]) where D is the post-P2 iterate.
    """
    X = _check_square(X)
    n = X.shape[0]
    if check_nonneg and np.any(X < 0):
        raise DataError("SDSN input must be nonnegative (S:251)")
    if scale:
        m = X.max()
        if m == 0.0:
            D = np.full((n, n), 1.0 / n)
            return (D, 0, []) if return_gammas else (D, 0)
        s = (theta / 2.0) / m
        Y = s * X
    else:
        Y = X.copy()
    gammas = []
    j = 0
    while True:
        r = Y.sum(axis=1)
        c = Y.sum(axis=0)
        S = r.sum()
        g = S / n - 1.0
        gammas.append(g)
        a = (1.0 / n + S / (n * n)) - r / n
        b = -c / n
        # Y = max(0, (Y + a) + b), evaluated in place (same operations in the same order,
        # bit-identical to the out-of-place expression; Y is this function's own copy)
        np.add(Y, a[:, None], out=Y)
        np.add(Y, b[None, :], out=Y)
        np.maximum(Y, 0.0, out=Y)
        j += 1
        if sdsn_fixed > 0:
            if j == sdsn_fixed:
                break
        elif (j - 1 >= 1 and g <= gamma_th) or j == sdsn_max:
            break
    return (Y, j, gammas) if return_gammas else (Y, j)


def sdsn_fp32(X, theta, gamma_th=1e-3, sdsn_max=1000, sdsn_fixed=0, scale=True, return_gammas=False):
    """SDSN (Alg. 2) with the iterate STORED IN FP32 — the emulated-rounding diagnostic
    reference of SURVEY §8(c) ("Rounding helpers"), for the paper's FP32 step 6.

    Same steps and grouping as `sdsn`; only the storage precision of Y differs (R9, R11, R13):
      Y⁰ = fl32(s·X), s = (θ/2)/max X in FP64                         (step 1, R11)
      r, c, S: FP64 sums of the FP32 values                            (R13)
      a_i = fl32((1/n + S/n²) − r_i/n),  b_j = fl32(−c_j/n)            (FP64, rounded once, R9)
      Y ← max(0, fl32(fl32(Y + a_i) + b_j))                            (step 6, FP32 adds)
    γ_j = S_j/n − 1 in FP64; stopping rule as `sdsn` (R5).  Input X: values representable in FP32.
    Returns (D as float64 holding FP32 values, passes[, gammas]).
    """
    X = _check_square(X)
    n = X.shape[0]
    if scale:
        m = X.max()
        if m == 0.0:
            D = np.full((n, n), np.float32(1.0 / n), dtype=np.float64)
            return (D, 0, []) if return_gammas else (D, 0)
        s = (theta / 2.0) / m
        Y = (s * X).astype(np.float32)
    else:
        Y = X.astype(np.float32)
    gammas = []
    j = 0
    while True:
        Y64 = Y.astype(np.float64)
        r = Y64.sum(axis=1)
        c = Y64.sum(axis=0)
        S = r.sum()
        g = S / n - 1.0
        gammas.append(g)
        a = ((1.0 / n + S / (n * n)) - r / n).astype(np.float32)
        b = (-c / n).astype(np.float32)
        np.add(Y, a[:, None], out=Y)                    # float32 + float32 → float32 (RNE)
        np.add(Y, b[None, :], out=Y)
        np.maximum(Y, np.float32(0.0), out=Y)
        j += 1
        if sdsn_fixed > 0:
            if j == sdsn_fixed:
                break
        elif (j - 1 >= 1 and g <= gamma_th) or j == sdsn_max:
            break
    D = Y.astype(np.float64)
    return (D, j, gammas) if return_gammas else (D, j)


def dsn_fixed(X, iters):
    """DSN with a fixed number of P2∘P1 rounds and no θ-scaling (DSPFP)."""
    D, _ = sdsn(X, theta=2.0, sdsn_fixed=iters, scale=False, check_nonneg=False)
    return D


# --------------------------------------------------------------------------------------
# Alg. 1 FRAM
# --------------------------------------------------------------------------------------
def fram(A, B, K=None, lam=1.0, theta=10.0, alpha=0.95, gamma_th=1e-3, delta_th=1e-4,
         max_outer=100, sdsn_max=1000, sdsn_fixed=0, X0=None, replay=None, scale=True,
         keep_trace=False, on_iter=None):
    """FRAM — Algorithm 1, FP64 throughout.

    O1-O2 precondition (steps 2-3); O3 N⁽⁰⁾ = X0 or 11ᵀ/n (R1); do-while outer loop (R2):
      G = A'NÃ' + λK' (step 5); D = SDSN(G, θ) (step 6);
      N ← (1−α)N + αD (step 7, unfused, R15); δ = ‖N_new − N‖_F/‖N_new‖_F (step 8, R14);
      stop if δ ≤ δ_th (step 4) or t = max_outer (R16).
    Step 10: perm = LAP_max(N) (R17).
    `replay`: per-outer-iteration SDSN pass counts to replay (parity harness):
      exactly len(replay) outer iterations run, pass t uses replay[t-1] passes.
    `on_iter(t, N, k_t, δ_t)`: optional observer called after each outer iteration.
    Returns a dict with N, perm, outer_iters, passes, deltas, converged, c and (keep_trace) Ns.
    """
    from .lap import lap_max

    Ap, Bp, Kp, c = precondition(A, B, K)
    n = Ap.shape[0]
    N = np.full((n, n), 1.0 / n) if X0 is None else np.array(X0, dtype=np.float64)
    passes, deltas, Ns = [], [], []
    converged = False
    T = len(replay) if replay is not None else max_outer
    t = 0
    for t in range(1, T + 1):
        G = gradient(Ap, N, Bp, Kp, lam)
        fixed = int(replay[t - 1]) if replay is not None else sdsn_fixed
        D, k = sdsn(G, theta, gamma_th, sdsn_max, fixed, scale, check_nonneg=False)
        N_new = (1.0 - alpha) * N + alpha * D
        delta = np.linalg.norm(N_new - N) / np.linalg.norm(N_new)
        N = N_new
        passes.append(k)
        deltas.append(float(delta))
        if keep_trace:
            Ns.append(N.copy())
        if on_iter is not None:          # observer only (checkpointing long runs); no arithmetic
            on_iter(t, N, k, float(delta))
        if delta <= delta_th:
            converged = True
            if replay is None:
                break
    if replay is not None:
        converged = bool(deltas and deltas[-1] <= delta_th)
    perm = lap_max(N)
    out = dict(N=N, perm=perm, outer_iters=t, passes=passes, deltas=deltas,
               converged=converged, c=c)
    if keep_trace:
        out["Ns"] = Ns
    return out


# --------------------------------------------------------------------------------------
# Attributed graphs of unequal size (NEXT-2 / NEXT-3): K = F F̃ᵀ and padding
# to a common size with isolated zero-attribute nodes ("n = ñ for simplicity")
# --------------------------------------------------------------------------------------
def unary_from_features(F, Ft):
    """K = F F̃ᵀ  (Eq.(1): ⟨NᵀF, F̃⟩ = ⟨N, F F̃ᵀ⟩; the gradient's unary term λK).
    F: n1×d, F̃: n2×d → K: n1×n2.  Library matmul as one step."""
    F = np.asarray(F, np.float64)
    Ft = np.asarray(Ft, np.float64)
    if F.ndim != 2 or Ft.ndim != 2 or F.shape[1] != Ft.shape[1]:
        raise ValueError("F and F̃ must be n1×d and n2×d")
    return F @ Ft.T


def pad_attributed(A, B, F, Ft, m):
    """Pad G (n1 nodes) and G̃ (n2 nodes) to m ≥ max(n1, n2) nodes by appending isolated nodes with
    zero attributes (R30): A, Ã → m×m with zero rows/columns, K = F F̃ᵀ → m×m with zero padding."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    n1, n2 = A.shape[0], B.shape[0]
    if m < max(n1, n2):
        raise ValueError("m must be >= max(n1, n2)")
    Ap = np.zeros((m, m)); Ap[:n1, :n1] = A
    Bp = np.zeros((m, m)); Bp[:n2, :n2] = B
    Kp = None
    if F is not None:
        Kp = np.zeros((m, m)); Kp[:n1, :n2] = unary_from_features(F, Ft)
    return Ap, Bp, Kp


def fram_attributed(A, B, F, Ft, m, lam=1.0, **kw):
    """FRAM on padded attributed graphs (R30): solve the m×m problem, then report, for each of the
    n1 nodes of G, the matched node of G̃, or −1 when it is matched to a padding node."""
    n1, n2 = np.asarray(A).shape[0], np.asarray(B).shape[0]
    Ap, Bp, Kp = pad_attributed(A, B, F, Ft, m)
    out = fram(Ap, Bp, Kp, lam=lam, **kw)
    perm = out["perm"][:n1].copy()
    perm[perm >= n2] = -1
    out["perm_attr"] = perm
    return out


# --------------------------------------------------------------------------------------
# Evaluation (Eq.(1); matching error P:379; accuracy P:383)
# --------------------------------------------------------------------------------------
def objective(A, B, K, N, lam=1.0):
    """Φ(N) = ½⟨NᵀAN, Ã⟩ + λ⟨N, K⟩  (Eq.(1), with K = FF̃ᵀ so ⟨NᵀF,F̃⟩ = ⟨N,K⟩)."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    N = np.asarray(N, np.float64)
    v = 0.5 * np.sum((N.T @ A @ N) * B)
    if K is not None:
        v += lam * np.sum(N * np.asarray(K, np.float64))
    return float(v)


def objective_perm(A, B, K, perm, lam=1.0):
    """Φ(M) for the matching matrix M with M[i, perm[i]] = 1:  ½ Σ_ij A_ij Ã_{perm i, perm j} + λ Σ_i K_{i, perm i}."""
    perm = np.asarray(perm, dtype=np.int64)
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    v = 0.5 * np.sum(A * B[np.ix_(perm, perm)])
    if K is not None:
        v += lam * np.sum(np.asarray(K, np.float64)[np.arange(len(perm)), perm])
    return float(v)


def matching_error(A, B, perm, F=None, Ft=None):
    """½‖A − MÃMᵀ‖_F + ‖F − MF̃‖_F;  (MÃMᵀ)_ij = Ã_{perm i, perm j}, (MF̃)_i = F̃_{perm i}."""
    perm = np.asarray(perm, dtype=np.int64)
    e = 0.5 * np.linalg.norm(np.asarray(A, np.float64) - np.asarray(B, np.float64)[np.ix_(perm, perm)])
    if F is not None:
        e += np.linalg.norm(np.asarray(F, np.float64) - np.asarray(Ft, np.float64)[perm])
    return float(e)


def node_accuracy(perm, perm_true, mask=None):
    """n_c / n; `mask` restricts to inlier rows (R20)."""
    perm = np.asarray(perm)
    perm_true = np.asarray(perm_true)
    ok = perm == perm_true
    if mask is not None:
        ok = ok[np.asarray(mask, bool)]
    return float(ok.mean())
