"""Pins for the oracle's P1 / P2 / P3 / γ (§5.1; Lemma P:919-927)."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle.exact import affine_projection_kkt

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _spec():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_p1_matches_kkt_solve(rng, n):
    # P1 closed form vs the equality-constrained least-squares KKT solve;
    # asymmetric X exercises the asymmetric-case theorem (proof).
    for _ in range(5):
        X = rng.normal(size=(n, n)) * 3.0
        assert np.max(np.abs(oracle.p1_project(X) - affine_projection_kkt(X))) <= 1e-10


def test_p1_zero_and_idempotent(rng):
    s = _spec()
    assert np.array_equal(oracle.p1_project(np.zeros((2, 2))), np.array(s["p1_zero_n2"]["out"]))
    X = rng.random((7, 7))
    Y = oracle.p1_project(X)
    assert np.max(np.abs(oracle.p1_project(Y) - Y)) <= 1e-12
    assert np.max(np.abs(Y.sum(1) - 1)) <= 1e-12 and np.max(np.abs(Y.sum(0) - 1)) <= 1e-12


def test_p1_minus_p3_is_uniform(rng):
    # Lemma: P1(X) − P3(X) = 11ᵀ/n exactly in exact arithmetic.
    for n in (3, 6, 11):
        X = rng.normal(size=(n, n))
        assert np.max(np.abs(oracle.p1_project(X) - oracle.p3_project(X) - 1.0 / n)) <= 1e-12
        Z = oracle.p3_project(X)
        assert np.max(np.abs(Z.sum(0))) <= 1e-12 and np.max(np.abs(Z.sum(1))) <= 1e-12


def test_p1_large_n_sums(rng):
    # Row/column sums of P1 output equal 1 (checked with compensated sums, R22).
    import math
    X = rng.random((300, 300))
    Y = oracle.p1_project(X)
    assert max(abs(math.fsum(r) - 1) for r in Y) <= 1e-12
    assert max(abs(math.fsum(c) - 1) for c in Y.T) <= 1e-12


def test_p2_examples():
    s = _spec()["p2"]
    assert np.array_equal(oracle.p2_nonneg(np.array(s["in"], float)), np.array(s["out"], float))
    assert np.array_equal(oracle.p2_nonneg(-np.eye(3)), np.zeros((3, 3)))


def test_gamma_examples():
    for case in _spec()["gamma"]:
        assert abs(oracle.gamma(np.array(case["in"], float)) - case["out"]) <= 1e-15
    assert abs(oracle.gamma(2 * np.ones((5, 5)) / 5)) - 1.0 <= 1e-15
    assert oracle.gamma(np.eye(4)) == 0.0
