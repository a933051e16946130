"""Race and ordering stress in place of compute-sanitizer (closed on this GPU pool): every kernel whose
cross-CTA or cross-warp exchange is barrier-free (K4r, K4, K4c: tagged words / st.async + mbarrier;
K7c: record exchange; K8; the virtual-shard collectives) is re-run many times on the same input, from
freshly created handles and with other work in between, and must return BIT-IDENTICAL results every
time (any race on Alg. 2's row/column sums, or on the LAP records would show up as a
different rounding, a different pass count, or a hang — the tests run under a timeout).  Each run is
also held to the oracle, so a consistently wrong result cannot pass either."""
import numpy as np
import pytest
import torch

import oracle
import paper_2508_00887_b200 as fb
from synth import config_c2, config_c3_batch, random_nonneg, random_perm_matrix

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]
REPS = 12


def _g(x, dt=torch.float64):
    return torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


@pytest.mark.parametrize("n,prec,kernel", [(20, "fp64", 4), (500, "fp64", 4), (64, "fp32", 4), (500, "fp32", 2),
                                           (2048, "fp32", 2), (4096, "fp32", 2), (2048, "fp64", 1), (4096, "fp64", 1),
                                           (5000, "fp32", 1)])
def test_sdsn_repeat_bit_identical(n, prec, kernel, errlog):
    rng = np.random.Generator(np.random.PCG64(n))
    X = random_nonneg(rng, n, "sparse") + 0.1 * np.eye(n)
    dt = torch.float64 if prec == "fp64" else torch.float32
    Xg = _g(X, dt)
    noise = torch.rand(8 * 1024 * 1024, device="cuda")
    outs = []
    for r in range(REPS):
        h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, gamma_th=1e-3, sdsn_max=300))
        noise.mul_(1.0001)                                      # unrelated work between the runs
        D, k, gam = fb.fram_sdsn(h, Xg, prec)
        outs.append((D.clone(), k, tuple(gam)))
    D0, k0, g0 = outs[0]
    for D, k, gm in outs[1:]:
        assert k == k0 and gm == g0 and torch.equal(D, D0)
    ref = oracle.sdsn(Xg.double().cpu().numpy(), 10.0, sdsn_fixed=k0)[0] if prec == "fp64" else \
        oracle.sdsn_fp32(Xg.double().cpu().numpy(), 10.0, sdsn_fixed=k0)[0]
    e = float(np.max(np.abs(D0.double().cpu().numpy() - ref)))
    errlog("max|D-ref| (repeat test)", e, 1e-12 if prec == "fp64" else 3e-2 / n, n=n)
    assert e <= (1e-12 if prec == "fp64" else 3e-2 / n)


@pytest.mark.parametrize("n", [500, 4096, 9000])
def test_lap_repeat_bit_identical(n):
    rng = np.random.Generator(np.random.PCG64(50 + n))
    N = 0.5 * random_perm_matrix(rng, n) + 0.45 * random_perm_matrix(rng, n) + 0.05 * rng.random((n, n))
    Ng = _g(N)
    h = fb.fram_create(n)
    p0 = fb.fram_lap(h, Ng).clone()
    for _ in range(REPS // 2):
        assert torch.equal(fb.fram_lap(fb.fram_create(n), Ng), p0)
    assert np.array_equal(p0.cpu().numpy(), oracle.lap_max(N))


def test_batched_repeat_bit_identical():
    insts = config_c3_batch(300)
    st = lambda a: _g(np.stack([getattr(i, a) for i in insts]), torch.float32)
    A, B, K = st("A"), st("B"), st("K")
    h = fb.fram_create(64, schedule=fb.Schedule(theta=2.0))
    _, _, X0, p0, s0 = fb.fram_solve_batched(h, A, B, K, precision="tf32")
    for _ in range(4):
        _, _, X, p, s = fb.fram_solve_batched(h, A, B, K, precision="tf32")
        assert torch.equal(X, X0) and torch.equal(p, p0) and np.array_equal(s, s0)


def test_virtual_shards_repeat_bit_identical():
    inst = config_c2(7, n=512)
    outs = []
    for _ in range(4):
        h = fb.fram_create_sharded_virtual(512, 1.0, fb.Schedule(theta=inst.theta, max_outer=4), world=4)
        _, s, X, p = fb.fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")
        outs.append((X.clone(), p.clone(), s["passes"]))
    for X, p, ps in outs[1:]:
        assert torch.equal(X, outs[0][0]) and torch.equal(p, outs[0][1]) and ps == outs[0][2]
