"""GPU parity: K1 preconditioning + K2/K3 gradient GEMMs, K7 LAP, vs the oracle.

Gradient tolerances:
  FP64 mode: DMMA FP64 products, different association than the oracle ((A'N)Ã' vs A'(NÃ')):
    ≤ 1e-12 relative to max|G|.
  Mixed modes: the GPU computes fl_op(fl_op(N)·Ã'_op)·A'_op with FP32 accumulation.  We compare
    with an FP64 product of the SAME quantised operands (emulated with oracle.rounding), where the
    only differences are FP32 accumulation (≤ γ_n·u32 relative, γ_n ≈ n) and the rounding of the
    intermediate U (same rounding rule, possibly flipped by accumulation error: ≤ 1 ulp_op of U).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle.rounding import round_bf16, round_fp16, round_tf32
from paper_2508_00887_b200 import FramError, Schedule, fram_create, fram_gradient, fram_lap, FRAM_ERR_DATA
from synth import ba_graph, er_graph, random_perm_matrix

pytestmark = pytest.mark.gpu
RND = {"bf16": (round_bf16, 2.0 ** -8), "fp16": (round_fp16, 2.0 ** -11), "tf32": (round_tf32, 2.0 ** -11)}


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def _g(x, dt=torch.float64):
    return torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


def _inputs(n, seed, withK=False):
    rng = _rng(seed)
    A = er_graph(rng, n, 0.1, weighted=True) * 3.0
    B = er_graph(rng, n, 0.1, weighted=True) * 2.0
    K = rng.random((n, n)) * 0.5 if withK else None
    N = rng.random((n, n))
    N /= N.sum(1, keepdims=True)
    return A, B, K, N


@pytest.mark.parametrize("n", [7, 64, 200, 513, 1500, 4096])
@pytest.mark.parametrize("withK", [False, True])
def test_gradient_fp64(n, withK):
    A, B, K, N = _inputs(n, n, withK)
    h = fram_create(n, lam=0.7)
    G, c = fram_gradient(h, _g(A), _g(B), _g(K) if withK else None, _g(N), "fp64")
    Ap, Bp, Kp, co = oracle.precondition(A, B, K)
    Go = oracle.gradient(Ap, N, Bp, Kp, 0.7)
    assert c == co
    assert np.max(np.abs(G.cpu().numpy() - Go)) <= 1e-12 * np.abs(Go).max()


@pytest.mark.parametrize("prec", ["bf16", "fp16", "tf32"])
@pytest.mark.parametrize("n", [20, 128, 300, 1000])
def test_gradient_mixed(prec, n):
    A, B, K, N = _inputs(n, 100 + n, withK=True)
    h = fram_create(n, lam=1.0)
    G, c = fram_gradient(h, _g(A), _g(B), _g(K), _g(N), prec)
    rnd, uop = RND[prec]
    Ap, Bp, Kp, _ = oracle.precondition(A, B, K)
    Aq, Bq, Nq = rnd(Ap), rnd(Bp), rnd(N)
    U = Nq @ Bq                                      # exact-ish FP64 product of quantised operands
    Uq = rnd(U)
    Gref = Aq @ Uq + Kp
    # error sources: FP32 accumulation in both products + one operand-format rounding flip of U
    bound = (4 * n * 2.0 ** -24) * (np.abs(Aq) @ np.abs(Uq)).max() + uop * (np.abs(Aq) @ np.abs(U)).max() \
        + 4 * 2.0 ** -24 * np.abs(Kp).max()
    err = np.max(np.abs(G.cpu().numpy().astype(np.float64) - Gref))
    assert err <= bound, (err, bound)
    # and the mixed gradient is close to the FP64 one at the operand precision
    Go = oracle.gradient(Ap, N, Bp, Kp, 1.0)
    assert np.max(np.abs(G.cpu().numpy() - Go)) <= 8 * uop * np.abs(Go).max()


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
@pytest.mark.parametrize("n", [2500, 4096])
def test_gradient_mixed_multi_tile(prec, n):
    # more 128×256 tiles than SMs (200 and 512 tiles on 148 SMs): the persistent GEMM reuses both TMEM
    # accumulator buffers and wraps the mbarrier phases; same bound as test_gradient_mixed
    test_gradient_mixed(prec, n)


@pytest.mark.parametrize("n,kind", [(2100, "random"), (3000, "nearperm"), (5000, "nearperm"), (6000, "twoperm"),
                                    (9000, "twoperm"), (16384, "nearperm")])
def test_lap_cluster_sizes_bit_exact(n, kind):
    # 2048 < n ≤ 8192 runs the R17 Hungarian on a 4-CTA cluster (K7c: columns split over the CTAs,
    # records exchanged by st.async/mbarrier, u/p/way replicated), 8192 < n ≤ 16384 on an 8-CTA
    # cluster with each CTA's copy of u in global memory: bit-exact with the oracle
    rng = _rng(7000 + n)
    if kind == "random":
        N = rng.random((n, n))
    elif kind == "nearperm":
        N = 0.8 * random_perm_matrix(rng, n) + 0.2 * rng.random((n, n)) / n
    else:
        N = 0.5 * random_perm_matrix(rng, n) + 0.45 * random_perm_matrix(rng, n) + 0.05 * rng.random((n, n))
    h = fram_create(n)
    p = fram_lap(h, _g(N)).cpu().numpy()
    assert np.array_equal(p, oracle.lap_max(N))


def test_gradient_bf16_storage_input():
    # FRAM_DT_BF16 inputs (C5 stores A dense in BF16): same result as the FP64 copy of those values.
    n = 96
    A, B, K, N = _inputs(n, 5)
    Ab = torch.tensor(A, dtype=torch.bfloat16, device="cuda")
    Bb = torch.tensor(B, dtype=torch.bfloat16, device="cuda")
    h = fram_create(n)
    G1, c1 = fram_gradient(h, Ab, Bb, None, _g(N), "fp64")
    G2, c2 = fram_gradient(h, Ab.double(), Bb.double(), None, _g(N), "fp64")
    assert c1 == c2 and torch.equal(G1, G2)


def test_precondition_errors():
    n = 16
    A, B, _, N = _inputs(n, 3)
    h = fram_create(n)
    bad = A.copy()
    bad[0, 1] = -1.0
    bad[1, 0] = -1.0
    with pytest.raises(FramError) as e:
        fram_gradient(h, _g(bad), _g(B), None, _g(N), "bf16")
    assert e.value.status == FRAM_ERR_DATA
    asym = A.copy()
    asym[0, 1] += 1.0
    with pytest.raises(FramError):
        fram_gradient(h, _g(asym), _g(B), None, _g(N), "bf16")
    with pytest.raises(FramError):
        fram_gradient(h, _g(np.zeros((n, n))), _g(np.zeros((n, n))), None, _g(N), "bf16")
    nanm = A.copy()
    nanm[2, 2] = np.nan
    with pytest.raises(FramError):
        fram_gradient(h, _g(nanm), _g(B), None, _g(N), "fp64")


# ------------------------------------------------------------------ LAP (K7), bit-exact (R17)
@pytest.mark.parametrize("n", [1, 2, 7, 33, 100, 257, 1000])
@pytest.mark.parametrize("kind", ["random", "nearperm", "ties"])
def test_lap_bit_exact(n, kind):
    rng = _rng(1000 + n)
    if kind == "random":
        N = rng.random((n, n))
    elif kind == "nearperm":
        N = 0.9 * random_perm_matrix(rng, n) + 0.1 * rng.random((n, n)) / n
    else:
        N = rng.integers(0, 3, (n, n)).astype(np.float64)
    h = fram_create(n)
    p = fram_lap(h, _g(N)).cpu().numpy()
    assert np.array_equal(p, oracle.lap_max(N))


def test_lap_large_nearperm():
    n = 4096
    rng = _rng(4096)
    P = random_perm_matrix(rng, n)
    N = 0.8 * P + 0.2 * rng.random((n, n)) / n
    h = fram_create(n)
    p = fram_lap(h, _g(N)).cpu().numpy()
    assert np.array_equal(p, oracle.lap_max(N))
    assert np.array_equal(p, np.argmax(P, axis=1))
