"""Pins for the oracle LAP (Eq.(2); Hungarian P:316; R17)."""
import json
import os

import numpy as np
import pytest
from scipy.optimize import linear_sum_assignment

from oracle.lap import brute_force_max, lap_max, perm_score

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_examples():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        cases = json.load(f)["lap"]
    for c in cases:
        N = np.array(c["in"], float)
        perm = lap_max(N)
        assert list(perm) == c["perm"]
        assert abs(perm_score(N, perm) - c["score"]) <= 1e-15


def test_identity_and_ones():
    assert list(lap_max(np.eye(4))) == [0, 1, 2, 3]
    assert list(lap_max(np.ones((6, 6)))) == list(range(6))   # all-ties → identity ([M21])


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_brute_force(rng, n):
    for _ in range(40):
        N = rng.random((n, n))
        perm = lap_max(N)
        bp, bs = brute_force_max(N)
        assert abs(perm_score(N, perm) - bs) <= 1e-12
        assert np.array_equal(perm, bp)       # continuous random ⇒ unique optimum a.s.


@pytest.mark.parametrize("n", [10, 39, 120])
def test_library_score(rng, n):
    for kind in ("cont", "int"):
        N = rng.random((n, n)) if kind == "cont" else rng.integers(0, 4, (n, n)).astype(float)
        perm = lap_max(N)
        assert sorted(perm) == list(range(n))
        r, c = linear_sum_assignment(-N)
        assert abs(perm_score(N, perm) - N[r, c].sum()) <= 1e-9


def test_round_trip(rng):
    for n in (5, 50):
        p = rng.permutation(n)
        M = np.zeros((n, n))
        M[np.arange(n), p] = 1.0
        assert np.array_equal(lap_max(M), p)
        # scale/shift invariance of the argmax
        assert np.array_equal(lap_max(3.0 * M + 0.25), p)


def test_empty():
    assert lap_max(np.zeros((0, 0))).shape == (0,)
