"""Tests for the seeded input generators (lofp_inputs) and the stored batches (data/)."""
import math
import os

import numpy as np
import pytest

import lofp_inputs as li
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("idx,nbs", [(0, 15), (1, 30), (2, 93), (3, 92), (4, 126)])
def test_config_bs_counts(idx, nbs):
    c = li.config(idx)
    assert sum(len(l) for l in c.layers) == nbs
    for l, layer in enumerate(c.layers, start=1):
        for a, b, th, ph in layer:
            assert b == a + 1 and (a % 2 == 0) == (l % 2 == 1)
            assert 0 <= th < math.pi / 2 and 0 <= ph < 2 * math.pi
    assert int(c.S.sum()) == c.N


def test_determinism():
    a, b = li.config(2), li.config(2)
    assert a.layers == b.layers
    assert np.array_equal(a.draw_outputs(B=16), b.draw_outputs(B=16))


def test_all_outputs_count():
    for M, N in [(6, 3), (4, 4), (1, 5), (7, 0)]:
        T = li.all_outputs(M, N)
        assert len(T) == math.comb(M + N - 1, N)
        assert len({tuple(t) for t in T}) == len(T) and (T.sum(1) == N).all()


def test_samplers_valid(rng):
    T = li.uniform_subsets(16, 8, 100, rng)
    assert (T.sum(1) == 8).all() and T.max() == 1
    T, total = li.bounded_patterns(24, 12, 2, 200, rng)
    assert (T.sum(1) == 12).all() and T.max() <= 2
    # number of patterns = coefficient of x^12 in (1 + x + x^2)^24 (independent route)
    poly = np.array([1], dtype=object)
    for _ in range(24):
        poly = np.convolve(poly, np.array([1, 1, 1], dtype=object))
    assert total == poly[12] == 287134346
    src = list(range(0, 48, 2))
    T, total = li.displaced_patterns(64, src, 4, 50, rng)
    assert (T.sum(1) == 24).all() and T.max() == 1
    for t in T:
        pos = np.nonzero(t)[0]
        assert np.all(np.abs(pos - np.array(src)) <= 4)


def test_displaced_count_brute_force():
    rng = np.random.default_rng(0)
    src = [0, 2, 4]
    _, total = li.displaced_patterns(8, src, 2, 1, rng)
    import itertools
    brute = sum(1 for c in itertools.combinations(range(8), 3) if all(abs(c[i] - src[i]) <= 2 for i in range(3)))
    assert total == brute


@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4])
def test_stored_batches(idx):
    path = os.path.join(ROOT, "data", f"cfg{idx}.npz")
    if not os.path.exists(path):
        pytest.skip("batch file not generated")
    d = np.load(path)
    c = li.config(idx)
    T = d["T_literal"].astype(np.int32)
    assert T.shape == (c.batch, c.M) and np.array_equal(T, c.draw_outputs())
    if "T_cond" in d:
        Tc = d["T_cond"].astype(np.int32)
        assert Tc.shape == (c.batch, c.M) and (Tc.sum(1) == c.N).all()
        assert (d["P_cond"] <= d["cap"]).all() and (d["P_cond"] > 0).all()
        # spot-check the stored counts against the oracle
        sel = np.arange(0, c.batch, max(1, c.batch // 16))
        assert oracle.count_paths(c.M, c.layers, c.S, Tc[sel]) == [int(x) for x in d["P_cond"][sel]]
    sel = np.arange(0, len(T), max(1, len(T) // 16))
    assert oracle.count_paths(c.M, c.layers, c.S, T[sel]) == [int(x) for x in d["P_literal"][sel]]
