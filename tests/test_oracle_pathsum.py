"""Pins for oracle_path_sum (eq. (1)) and the light cones.

The path sum is pinned to the permanent formula (Ryser), to unitarity
over all outputs, to the depth<=2 single-path product (eq. 10), to
vacuum / identity / photon-number special cases, and its three prune modes to each
other (the paper's cone bounds and the cumulative box must never drop a valid path).
"""
import json
import math
import os

import numpy as np
import pytest

import lofp_inputs as li
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_lightcone_worked_example():
    g = json.load(open(os.path.join(GOLDEN, "lightcone_p164.json")))
    layers = li.clements_mesh(g["M"], g["D"], seed=0)
    past, fut = oracle.cone_sets(g["M"], layers, g["mode_1based"] - 1, g["segment"])
    assert sorted(np.nonzero(past)[0] + 1) == g["past_1based"]
    assert sorted(np.nonzero(fut)[0] + 1) == g["future_1based"]


@pytest.mark.parametrize("seed", range(12))
def test_pathsum_vs_ryser_random_nn(seed):
    rng = np.random.default_rng(seed)
    M = int(rng.integers(2, 8))
    D = int(rng.integers(0, 7))
    N = int(rng.integers(0, 5))
    layers = li.random_nn_circuit(M, D, rng, fill=0.8, reverse_prob=0.3)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    T = li.all_outputs(M, N)
    ref = oracle.amplitudes_permanent(M, layers, S, T)
    results = {}
    for prune in (oracle.PRUNE_NONE, oracle.PRUNE_CONE, oracle.PRUNE_BOX):
        a, leaves = oracle.path_sum(M, layers, S, T, prune=prune, return_leaves=True)
        assert np.abs(a - ref).max() < 1e-13, prune
        results[prune] = leaves
    # pruning never drops a valid path
    assert np.array_equal(results[0], results[1]) and np.array_equal(results[0], results[2])
    assert abs(np.sum(np.abs(ref) ** 2) - 1) < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_pathsum_non_nearest_neighbour(seed):
    """Prunes 0 and 1 do not assume adjacent pairs (the paper's cones are generic)."""
    rng = np.random.default_rng(50 + seed)
    M, D = 6, 3
    layers = []
    for _ in range(D):
        perm = rng.permutation(M)
        layers.append([(int(perm[2 * i]), int(perm[2 * i + 1]), float(rng.uniform(0, 1.5)), float(rng.uniform(0, 6)))
                       for i in range(int(rng.integers(1, 4)))])
    S = np.array([1, 0, 2, 0, 1, 0])
    T = li.all_outputs(M, 4)
    ref = oracle.amplitudes_permanent(M, layers, S, T)
    for prune in (0, 1):
        assert np.abs(oracle.path_sum(M, layers, S, T, prune=prune) - ref).max() < 1e-13


def test_config0_distribution():
    """BASELINE.json configs[0]: all 56 outputs, sum |a|^2 = 1, equal to Ryser."""
    c = li.config(0)
    T = c.draw_outputs()
    assert T.shape == (56, 6)
    a, leaves = oracle.path_sum(c.M, c.layers, c.S, T, return_leaves=True)
    ref = oracle.amplitudes_permanent(c.M, c.layers, c.S, T)
    assert np.abs(a - ref).max() < 1e-14
    assert abs(np.sum(np.abs(a) ** 2) - 1) < 1e-13
    assert int(leaves.sum()) == 9639


@pytest.mark.parametrize("case", range(4))
def test_paper_correctness_protocol(case):
    """four 6-mode inputs at depths 3..6, all outputs, sum p = 1 and TVD vs Ryser."""
    S, D = li.paper_correctness_inputs()[case]
    layers = li.clements_mesh(6, D, seed=1000 + case)
    T = li.all_outputs(6, sum(S))
    a = oracle.path_sum(6, layers, S, T)
    ref = oracle.amplitudes_permanent(6, layers, S, T)
    p, q = np.abs(a) ** 2, np.abs(ref) ** 2
    assert abs(p.sum() - 1) < 1e-12
    assert oracle.tvd(p, q) < 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_depth_le_two_single_path(seed):
    """Eq. (10): for D <= 2 a valid path is unique and the amplitude is the product of the
    BS elements along it.  The path is found here by propagating occupations BS by BS in
    Python (each BS output split determined by T through the layer-2 BS)."""
    rng = np.random.default_rng(200 + seed)
    M = 8
    layers = li.clements_mesh(M, 2, seed=seed)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=4):
        S[m] += 1
    T = li.all_outputs(M, 4)
    a, leaves = oracle.path_sum(M, layers, S, T, return_leaves=True)
    assert leaves.max() <= 1
    ref = oracle.amplitudes_permanent(M, layers, S, T)
    assert np.abs(a - ref).max() < 1e-13
    # explicit product for every reachable output
    for t, amp, lv in zip(T, a, leaves):
        # layer-2 BS (1,2),(3,4),(5,6) see (mid[k], mid[k+1]) -> (t[k], t[k+1]); modes 0 and 7 pass through
        mid = np.zeros(M, dtype=int)
        mid[0], mid[M - 1] = t[0], t[M - 1]
        prod = 1.0 + 0j
        ok = True
        for (p, q, th, ph) in layers[0]:  # layer 1 pairs (0,1),(2,3),..: output split fixed by mid
            n = S[p] + S[q]
            # mode p's layer-1 output is fixed by layer 2: mode 0 passes to the output; mode p>0 is the
            # lower port of layer-2 BS (p-1, p), whose input from above is known recursively
            if p == 0:
                mid[p] = t[0]
            else:
                mid[p] = t[p - 1] + t[p] - mid[p - 1]
            mid[q] = n - mid[p]
            if mid[p] < 0 or mid[q] < 0:
                ok = False
                break
            prod *= oracle.bs_element(th, ph, S[p], S[q], mid[p], mid[q])
        if ok:
            for (p, q, th, ph) in layers[1]:
                if mid[p] + mid[q] != t[p] + t[q]:
                    ok = False
                    break
                prod *= oracle.bs_element(th, ph, mid[p], mid[q], t[p], t[q])
        if ok and mid[M - 1] != t[M - 1]:
            ok = False
        if lv == 1:
            assert ok and abs(prod - amp) < 1e-13
        else:
            assert amp == 0


def test_special_cases(rng):
    c = li.config(1)
    # vacuum -> 1
    a = oracle.path_sum(c.M, c.layers, np.zeros(c.M, dtype=int), np.zeros((1, c.M), dtype=int))
    assert a[0] == 1
    # theta = 0 everywhere: identity -> delta_{S,T}
    zl = [[(p, q, 0.0, ph) for (p, q, th, ph) in l] for l in c.layers]
    T = np.stack([c.S, np.roll(c.S, 1), li.uniform_subsets(c.M, c.N, 1, rng)[0]])
    a = oracle.path_sum(c.M, zl, c.S, T)
    assert a[0] == 1 and a[1] == 0 and (a[2] == 0 or np.array_equal(T[2], c.S))
    # photon number mismatch -> exact 0
    T = np.zeros((1, c.M), dtype=int)
    T[0, :3] = 1
    assert oracle.path_sum(c.M, c.layers, c.S, T)[0] == 0
    # D = 0 -> delta
    assert oracle.path_sum(4, [], [1, 0, 2, 0], [[1, 0, 2, 0], [0, 1, 2, 0]]).tolist() == [1, 0]


def test_reversed_pair_is_swapped_phase(rng):
    """Reading R4: a pair listed as (b, a, theta, phi) equals (a, b, theta, pi - phi)."""
    M = 6
    layers = li.random_nn_circuit(M, 4, rng)
    rev = [[(q, p, th, ph) for (p, q, th, ph) in l] for l in layers]
    canon = [[(p, q, th, math.pi - ph) for (p, q, th, ph) in l] for l in layers]
    S = [1, 0, 1, 1, 0, 0]
    T = li.all_outputs(M, 3)
    assert np.abs(oracle.path_sum(M, rev, S, T) - oracle.path_sum(M, canon, S, T)).max() < 1e-14


@pytest.mark.parametrize("seed", range(8))
def test_nonlocal_pathsum_vs_ryser(seed):
    """Non-local pairs (NEXT-4): the oracle's path sum with the paper's cone bounds (P:164,
    prune 1) and with no prune agree with each other and with Ryser."""
    rng = np.random.default_rng(800 + seed)
    M = int(rng.integers(3, 7))
    D = int(rng.integers(1, 5))
    N = int(rng.integers(1, 5))
    layers = li.random_nonlocal_circuit(M, D, rng)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    T = li.all_outputs(M, N)
    a1, l1 = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_CONE, return_leaves=True)
    a0, l0 = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_NONE, return_leaves=True)
    ref = oracle.amplitudes_permanent(M, layers, S, T)
    assert np.abs(a1 - ref).max() < 1e-13
    assert np.abs(a0 - ref).max() < 1e-13
    assert np.array_equal(l0, l1)  # the cone bound never drops a valid path
    assert abs(np.sum(np.abs(a1) ** 2) - 1) < 1e-13
