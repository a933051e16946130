"""Generator sanity (data only): symmetry, sizes, planted orientation (R18)."""
import numpy as np

from synth import config_c1, config_c2, config_c3_instance, ba_graph


def _check_planted(inst, An=None):
    A, B, s = inst.A, inst.B, inst.perm_true
    assert np.array_equal(A, A.T) and np.array_equal(B, B.T)
    assert np.all(A >= 0) and np.all(B >= 0)
    if An is not None:
        assert np.array_equal(B[np.ix_(s, s)], An)


def test_c1():
    inst = config_c1(0)
    assert inst.n == 20 and inst.K is None and inst.theta == 10.0
    _check_planted(inst)
    assert np.all(np.diag(inst.A) == 0)
    # deterministic
    assert np.array_equal(config_c1(0).B, inst.B)
    # the noise is a small number of toggles
    E = np.triu(inst.A, 1).sum()
    diff = np.triu(np.abs(inst.A - inst.B[np.ix_(inst.perm_true, inst.perm_true)]), 1).sum()
    assert diff == round(0.05 * E)


def test_c2_small():
    inst = config_c2(0, n=120)
    _check_planted(inst)
    assert inst.A.max() <= 1.0


def test_c3():
    inst = config_c3_instance(np.random.SeedSequence(3).spawn(2)[1])
    assert inst.n == 64 and inst.K.shape == (64, 64) and inst.theta == 2.0
    assert inst.inlier_mask.sum() == 64 - 6
    assert np.allclose(np.diag(inst.A), 1.0)


def test_ba_edges():
    rng = np.random.Generator(np.random.PCG64(0))
    A = ba_graph(rng, 200, 5)
    assert np.triu(A, 1).sum() == 5 * (200 - 5)
    assert np.array_equal(A, A.T)
