"""GPU parity at config C5's full size (n = 16384), in the kernels and launch configuration the C5 path
uses on one GPU: the BF16 gradient GEMMs (K2/K3, BF16-stored inputs as C5 stores A) on sampled
output columns, and the streaming FP32 SDSN (K4, 148 CTAs, 8 vectors per lane) against the
FP32-stored oracle over a few whole passes.  (The LAP at n = 16384 is in test_gpu_kernels.py.)

Sampled gradient columns: G[:, j] = A'_q · fl_bf16(N_q · Ã'_q[:, j]) needs only matrix-vector products,
so the oracle computes the sampled columns one by one (Alg. 1 step 5; R12 rounding).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle.rounding import round_bf16
from paper_2508_00887_b200 import Schedule, fram_create, fram_gradient, fram_sdsn
from synth import config_c5, random_nonneg

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1800)]
N5 = 16384
U32 = 2.0 ** -24


@pytest.fixture(scope="module")
def c5():
    return config_c5(0)


def test_c5_gradient_sampled_columns_bf16(c5, errlog):
    n = N5
    rng = np.random.Generator(np.random.PCG64(5))
    N = rng.random((n, n))
    N /= N.sum(1, keepdims=True)
    h = fram_create(n, lam=1.0)
    Ag = torch.tensor(c5.A, dtype=torch.bfloat16, device="cuda")      # exact: the C5 values are BF16
    Bg = torch.tensor(c5.B, dtype=torch.bfloat16, device="cuda")
    G, c = fram_gradient(h, Ag, Bg, None, torch.tensor(N, device="cuda"), "bf16")
    A = c5.A.astype(np.float64)
    B = c5.B.astype(np.float64)
    Ap, Bp, _, co = oracle.precondition(A, B, None)
    assert c == co
    del A, B
    Aq, Bq, Nq = round_bf16(Ap), round_bf16(Bp), round_bf16(N)
    del Ap, Bp, N
    cols = np.concatenate([[0, 1, n - 1], rng.choice(np.arange(2, n - 1), size=5, replace=False)])
    Gs = G[:, torch.tensor(cols, device="cuda")].double().cpu().numpy()
    absA = np.abs(Aq)
    worst = 0.0
    for k, j in enumerate(cols):
        u = Nq @ Bq[:, j]                              # FP64 product of the quantised operands
        uq = round_bf16(u)
        g = Aq @ uq
        bound = 4 * n * U32 * float((absA @ np.abs(uq)).max()) + 2.0 ** -8 * float((absA @ np.abs(u)).max())
        err = float(np.max(np.abs(Gs[:, k] - g)))
        worst = max(worst, err / bound)
        assert err <= bound, (j, err, bound)
    errlog("c5 gradient sampled cols err/bound", worst, 1.0, n=n, cols=len(cols))


@pytest.mark.parametrize("k", [3])
def test_c5_sdsn_fp32_full_passes(k, errlog):
    n = N5
    X = random_nonneg(np.random.Generator(np.random.PCG64(16384)), n, "sparse").astype(np.float32)
    h = fram_create(n, schedule=Schedule(theta=10.0, sdsn_fixed=k))
    D, kk, gam = fram_sdsn(h, torch.tensor(X, device="cuda"), "fp32")
    assert kk == k
    Dg = D.cpu().numpy()
    del D
    D32, _, g32 = oracle.sdsn_fp32(X.astype(np.float64), 10.0, sdsn_fixed=k, return_gammas=True)
    e32 = float(np.max(np.abs(Dg.astype(np.float64) - D32)))
    errlog("c5 sdsn max|D_gpu-D_fp32emu|*n", e32 * n, 3e-2, n=n, k=k)
    assert e32 * n <= 3e-2                            # test_gpu_sdsn.py's TOL_EMU (× 1/n)
    tg = 64 * U32 * (1.0 + max(g32))
    assert np.max(np.abs(np.array(gam[:k]) - np.array(g32[:k]))) <= tg
    # invariants after the last pass (R22): row and column sums ≥ 1 − O(u), equal clamped mass
    r = Dg.astype(np.float64).sum(1)
    c = Dg.astype(np.float64).sum(0)
    assert r.min() >= 1.0 - 1e-3 and c.min() >= 1.0 - 1e-3
