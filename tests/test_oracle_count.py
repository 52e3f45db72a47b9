"""Pins for oracle_count_paths (reading R6) and oracle_reachable (reading R5).

Both are pinned to brute force: the number of leaves the unpruned path sum reaches
(every BS split enumerated, only the final check against T) on many random small
nearest-neighbour circuits, including partial layers and reversed pairs.
"""
import math

import numpy as np
import pytest

import lofp_inputs as li
import oracle


@pytest.mark.parametrize("seed", range(40))
def test_count_and_reachability_vs_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    M = int(rng.integers(1, 8))
    D = int(rng.integers(0, 7))
    N = int(rng.integers(0, 6))
    layers = li.random_nn_circuit(M, D, rng, fill=float(rng.uniform(0.5, 1.0)), reverse_prob=0.3)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    T = li.all_outputs(M, N)
    if len(T) > 120:
        T = T[rng.choice(len(T), 120, replace=False)]
    _, leaves = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_NONE, return_leaves=True)
    counts = oracle.count_paths(M, layers, S, T)
    assert [int(x) for x in leaves] == counts
    assert np.array_equal(oracle.reachable(M, layers, S, T), leaves > 0)
    # the box-pruned sum reaches no dead end and no more leaves
    _, lb = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_BOX, return_leaves=True)
    assert np.array_equal(lb, leaves)


def test_count_depth_le_two_is_zero_or_one(rng):
    for D in (1, 2):
        layers = li.clements_mesh(10, D, seed=D)
        S = np.array([1, 0, 2, 0, 0, 1, 1, 0, 0, 1])
        T = li.all_outputs(10, 6)[::7]
        assert set(oracle.count_paths(10, layers, S, T)) <= {0, 1}


def test_count_photon_mismatch_and_vacuum():
    layers = li.clements_mesh(6, 4, seed=1)
    assert oracle.count_paths(6, layers, [1, 1, 0, 0, 0, 0], [[1, 0, 0, 0, 0, 0]]) == [0]
    assert oracle.count_paths(6, layers, [0] * 6, [[0] * 6]) == [1]


def test_count_single_photon_is_number_of_walks():
    """One photon: a valid path is a walk through the mesh; with full brickwork layers the
    photon either stays or crosses at every BS it meets, so paths from mode s to mode t in
    D layers number the walks of a known lattice — brute-force them independently."""
    M, D = 8, 5
    pairs = li.clements_pairs(M, D)
    layers = li.clements_mesh(M, D, seed=0)
    for s in range(M):
        # count walks by dynamic programming over layers (different code from the oracle)
        ways = np.zeros(M, dtype=object)
        ways[s] = 1
        for pl in pairs:
            nxt = ways.copy()
            for a, b in pl:
                nxt[a] = ways[a] + ways[b]
                nxt[b] = ways[a] + ways[b]
            ways = nxt
        S = np.eye(M, dtype=int)[s]
        T = np.eye(M, dtype=int)
        assert oracle.count_paths(M, layers, S, T) == [int(w) for w in ways]


def test_count_large_config_runs():
    """The counter handles the big configs (exact 128-bit counts)."""
    c = li.config(3)
    T = c.draw_outputs(B=8)
    cnt = oracle.count_paths(c.M, c.layers, c.S, T)
    assert all(x is not None for x in cnt)
    assert max(cnt) > 10 ** 10
