"""The W > 1 row-sharded path (config C5's partition) on ONE GPU: a virtual-shard group
(fram_create_sharded_virtual) runs W ranks of the unchanged sharded solve, one host thread and stream
each, with the NCCL all-gather / all-reduce replaced by fixed-order device copies and sums.

This executes everything a real W-GPU solve does per rank — row offsets of A, K, N, G; the K-blocked
3-D TMA (mixed) / blocked cp.async (FP64) GEMM operand reading W gathered Uᵀ blocks in place; the
row-block K4s SDSN whose column sums and mass are all-reduced every pass; the rank-identical stop
decisions (γ, δ) from reduced values; the N all-gather and a LAP on every rank.

Acceptance as for W = 1 (Alg. 1, steps 5-8 partitioned by rows):
  FP64: max|N_W⁽ᵗ⁾ − N_oracle⁽ᵗ⁾| ≤ 1e-9 per outer iteration with the oracle replaying the pass counts,
        the same pass counts as the W = 1 sharded solve, and ≤ 1e-12 from it (only the FP64 summation
        order of the column sums differs: per-rank CTA partials, then ranks in order);
  mixed: |ΔΦ|/Φ ≤ 1e-3 and |Δacc| ≤ 0.5 pp against W = 1; LAP bit-exact on the returned N.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2508_00887_b200 as fb
from synth import config_c2

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


def _g(x, dt=torch.float64):
    return torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


def _solve(inst, W, prec, K=None, **kw):
    dt = torch.float64 if prec == "fp64" else torch.float32
    sch = fb.Schedule(theta=inst.theta, flags=fb.FLAG_TRACE | fb.FLAG_CHECK_SYMMETRY, **kw)
    if W == 0:                                             # the real one-rank NCCL sharded handle
        h = fb.fram_create_sharded(inst.n, 1.0, sch, fb.fram_get_unique_id(), 0, 1)
    else:
        h = fb.fram_create_sharded_virtual(inst.n, 1.0, sch, world=W)
    return fb.fram_solve(h, _g(inst.A, dt), _g(inst.B, dt), None if K is None else _g(K, dt), precision=prec)


@pytest.mark.parametrize("n,W", [(256, 2), (256, 4), (256, 8), (520, 8), (1000, 4), (2048, 8)])
def test_virtual_shards_fp64_vs_oracle_and_w1(n, W, errlog):
    inst = config_c2(3, n=n)
    max_outer = 4 if n >= 1000 else 100
    st1, s1, X1, p1 = _solve(inst, 0, "fp64", max_outer=max_outer)
    stW, sW, XW, pW = _solve(inst, W, "fp64", max_outer=max_outer)
    assert sW["sdsn_kernel"] == 3
    assert sW["passes"] == s1["passes"] and sW["outer_iters"] == s1["outer_iters"]
    d1 = float(np.max(np.abs(XW.cpu().numpy() - X1.cpu().numpy())))
    errlog("max|N_W-N_W1|", d1, 1e-12, W=W, n=n)
    assert d1 <= 1e-12
    ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta, replay=sW["passes"], keep_trace=True)
    e = float(np.max(np.abs(XW.cpu().numpy() - ref["N"])))
    errlog("max|N_W-N_oracle|", e, 1e-9, W=W, n=n)
    assert e <= 1e-9
    assert np.max(np.abs(np.array(sW["deltas"]) - np.array(ref["deltas"]))) <= 1e-9
    assert np.array_equal(pW.cpu().numpy(), ref["perm"])
    # per outer iteration: a replayed prefix of t iterations on the virtual group
    t = max(1, len(sW["passes"]) // 2)
    _, _, Xt, _ = _solve(inst, W, "fp64", replay=sW["passes"][:t])
    et = float(np.max(np.abs(Xt.cpu().numpy() - ref["Ns"][t - 1])))
    errlog("max|N_W-N_oracle|", et, 1e-9, W=W, n=n, t=t)
    assert et <= 1e-9


def test_virtual_shards_fp64_unary_term(errlog):
    inst = config_c2(4, n=384)
    K = np.random.Generator(np.random.PCG64(8)).random((inst.n, inst.n)) * 0.2
    _, sW, XW, pW = _solve(inst, 4, "fp64", K=K, max_outer=5)
    ref = oracle.fram(inst.A, inst.B, K, theta=inst.theta, replay=sW["passes"])
    e = float(np.max(np.abs(XW.cpu().numpy() - ref["N"])))
    errlog("max|N_W-N_oracle|", e, 1e-9, W=4, n=inst.n)
    assert e <= 1e-9
    assert np.array_equal(pW.cpu().numpy(), ref["perm"])


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_virtual_shards_mixed_vs_w1(prec, W, errlog):
    inst = config_c2(5, n=512)                             # (n/W) % 64 == 0 for the tcgen05 row blocks
    _, s1, X1, p1 = _solve(inst, 0, prec)
    _, sW, XW, pW = _solve(inst, W, prec)
    phi1 = oracle.objective_perm(inst.A, inst.B, None, p1.cpu().numpy())
    phiW = oracle.objective_perm(inst.A, inst.B, None, pW.cpu().numpy())
    errlog("|dPhi|/Phi (W vs 1)", abs(phiW - phi1) / abs(phi1), 1e-3, W=W)
    assert abs(phiW - phi1) <= 1e-3 * abs(phi1)
    a1 = oracle.node_accuracy(p1.cpu().numpy(), inst.perm_true)
    aW = oracle.node_accuracy(pW.cpu().numpy(), inst.perm_true)
    assert abs(aW - a1) <= 0.005
    assert np.array_equal(pW.cpu().numpy(), oracle.lap_max(XW.cpu().numpy()))


def test_virtual_shards_errors_do_not_hang():
    inst = config_c2(0, n=256)
    Z = np.zeros((256, 256))
    h = fb.fram_create_sharded_virtual(256, 1.0, fb.Schedule(theta=10.0), world=4)
    with pytest.raises(fb.FramError) as e:                 # c = 0 on every rank
        fb.fram_solve(h, _g(Z), _g(Z), precision="fp64")
    assert e.value.status == fb.FRAM_ERR_DATA
    bad = inst.A.copy()
    bad[200, 3] = np.nan                                  # only rank 3's rows are bad: the reduced scan fails all
    with pytest.raises(fb.FramError) as e:
        fb.fram_solve(h, _g(bad), _g(inst.B), precision="fp64")
    assert e.value.status == fb.FRAM_ERR_DATA
    with pytest.raises(fb.FramError) as e:
        fb.fram_sdsn(h, _g(np.eye(256)), "fp64")
    assert e.value.status == fb.FRAM_ERR_USAGE
    _, s, X, p = fb.fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")      # still usable
    assert sorted(p.cpu().numpy()) == list(range(256))


def test_virtual_shards_host_buffers_match_device():
    inst = config_c2(6, n=256)
    h = fb.fram_create_sharded_virtual(256, 1.0, fb.Schedule(theta=inst.theta, max_outer=5), world=2)
    _, s1, X1, p1 = fb.fram_solve(h, _g(inst.A), _g(inst.B), precision="fp64")
    _, s2, X2, p2 = fb.fram_solve(h, np.ascontiguousarray(inst.A), np.ascontiguousarray(inst.B), precision="fp64")
    assert isinstance(X2, np.ndarray) and np.array_equal(X1.cpu().numpy(), X2)
    assert np.array_equal(p1.cpu().numpy(), p2) and s1["passes"] == s2["passes"]
