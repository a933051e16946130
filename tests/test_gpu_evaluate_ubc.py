"""NEXT-2: the attributed, fully connected keypoint-graph regime of the paper's ubc(2000)
task (Fig. 3; graphs from images P:1047: Euclidean-distance edges, node attributes, θ = 2)
on the synthetic stand-in synth.config_ubc, and the device-side evaluation K9 (fram_evaluate: the
matching error of P:379 and Φ(M) of Eq.(1)) against the oracle's matching_error / objective_perm.
"""
import functools
import json
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2508_00887_b200 as fb
from synth import config_c2, config_ubc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "ubc2000_oracle.json")


def _g(x, dt=torch.float64):
    return torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")


@pytest.mark.parametrize("n,d,dt", [(7, 3, torch.float64), (300, 128, torch.float64), (513, 64, torch.float32),
                                    (1000, 0, torch.float64)])
def test_evaluate_matches_oracle(n, d, dt, errlog):
    rng = np.random.Generator(np.random.PCG64(n + d))
    A = rng.random((n, n)); A = A + A.T
    B = rng.random((n, n)); B = B + B.T
    F, Ft = (rng.random((n, d)), rng.random((n, d))) if d else (None, None)
    if dt == torch.float32:                                 # the oracle sees the FP32 values exactly
        A, B = (x.astype(np.float32).astype(np.float64) for x in (A, B))
        F, Ft = (x.astype(np.float32).astype(np.float64) for x in (F, Ft))
    perm = rng.permutation(n).astype(np.int32)
    h = fb.fram_create(n, lam=0.7)
    r = fb.fram_evaluate(h, _g(A, dt), _g(B, dt), _g(perm, torch.int32), None if F is None else _g(F, dt),
                         None if Ft is None else _g(Ft, dt))
    me = oracle.matching_error(A, B, perm, F, Ft)
    K = None if F is None else oracle.unary_from_features(F, Ft)
    phi = oracle.objective_perm(A, B, K, perm, lam=0.7)
    errlog("|err_gpu-err_oracle|/err", abs(r["matching_error"] - me) / me, 1e-12)
    assert abs(r["matching_error"] - me) <= 1e-12 * me
    assert abs(r["phi"] - phi) <= 1e-12 * abs(phi)
    # host buffers give the same bits; an invalid perm is a data error
    r2 = fb.fram_evaluate(h, np.ascontiguousarray(A.astype(np.float32 if dt == torch.float32 else np.float64)),
                          np.ascontiguousarray(B.astype(np.float32 if dt == torch.float32 else np.float64)), perm,
                          None if F is None else np.ascontiguousarray(F.astype(np.float32 if dt == torch.float32 else np.float64)),
                          None if Ft is None else np.ascontiguousarray(Ft.astype(np.float32 if dt == torch.float32 else np.float64)))
    assert r2 == r
    bad = perm.copy()
    bad[0] = n
    with pytest.raises(fb.FramError) as e:
        fb.fram_evaluate(h, _g(A, dt), _g(B, dt), _g(bad, torch.int32))
    assert e.value.status == fb.FRAM_ERR_DATA


@pytest.mark.parametrize("n", [300, 640])
def test_ubc_fp64_replay_and_mixed(n, errlog):
    inst = config_ubc(1, n=n)
    F, Ft = inst.meta["F"], inst.meta["Ft"]
    h = fb.fram_create(n, schedule=fb.Schedule(theta=2.0))
    st, s64, X, perm = fb.fram_solve_attributed(h, _g(inst.A), _g(inst.B), _g(F), _g(Ft), precision="fp64")
    ref = oracle.fram_attributed(inst.A, inst.B, F, Ft, n, theta=2.0, replay=s64["passes"])
    e = float(np.max(np.abs(X.cpu().numpy() - ref["N"])))
    errlog("max|N_gpu-N_oracle|", e, 1e-9, n=n)
    assert e <= 1e-9
    assert np.array_equal(perm.cpu().numpy(), ref["perm_attr"])
    free = oracle.fram_attributed(inst.A, inst.B, F, Ft, n, theta=2.0)
    assert free["passes"] == s64["passes"]
    me_o = oracle.matching_error(inst.A, inst.B, free["perm_attr"], F, Ft)
    for prec in ("tf32", "bf16"):
        _, sm, Xm, pm = fb.fram_solve_attributed(h, _g(inst.A), _g(inst.B), _g(F), _g(Ft), precision=prec)
        p = pm.cpu().numpy()
        ev = fb.fram_evaluate(h, _g(inst.A), _g(inst.B), _g(p, torch.int32), _g(F), _g(Ft))
        phi_o = oracle.objective_perm(inst.A, inst.B, oracle.unary_from_features(F, Ft), free["perm_attr"])
        errlog("|dPhi|/Phi", abs(ev["phi"] - phi_o) / phi_o, 1e-3, prec=prec, n=n)
        assert abs(ev["phi"] - phi_o) <= 1e-3 * phi_o
        assert abs(oracle.node_accuracy(p, inst.perm_true) - oracle.node_accuracy(free["perm_attr"], inst.perm_true)) <= 0.005
        errlog("matching error gpu vs oracle solve", ev["matching_error"], me_o, prec=prec, n=n)


@functools.lru_cache(None)
def _gold():
    with open(GOLD) as f:
        return json.load(f)


@pytest.mark.parametrize("prec", ["fp64", "tf32", "bf16"])
def test_ubc2000_vs_oracle_golden(prec, errlog):
    # full size n = 2000 against the oracle's full solve (tests/golden/ubc2000_oracle.json)
    gold = _gold()
    inst = config_ubc(0, n=2000)
    F, Ft = inst.meta["F"], inst.meta["Ft"]
    h = fb.fram_create(2000, schedule=fb.Schedule(theta=2.0))
    st, s, X, perm = fb.fram_solve_attributed(h, _g(inst.A), _g(inst.B), _g(F), _g(Ft), precision=prec)
    p = perm.cpu().numpy()
    ev = fb.fram_evaluate(h, _g(inst.A), _g(inst.B), _g(p, torch.int32), _g(F), _g(Ft))
    errlog("|dPhi|/Phi", abs(ev["phi"] - gold["phi_perm"]) / gold["phi_perm"], 1e-3, prec=prec)
    assert abs(ev["phi"] - gold["phi_perm"]) <= 1e-3 * gold["phi_perm"]
    acc = oracle.node_accuracy(p, inst.perm_true)
    assert abs(acc - gold["accuracy"]) <= 0.005
    if prec == "fp64":
        assert s["passes"] == gold["passes"]
        assert p.tolist() == gold["perm"]
        assert abs(ev["matching_error"] - gold["matching_error"]) <= 1e-9 * gold["matching_error"]
