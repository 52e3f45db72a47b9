"""Pins for the oracle permanents and circuit unitary."""
import itertools
import math

import numpy as np
import pytest

import lofp_inputs as li
import oracle


def perm_definition(A):
    n = A.shape[0]
    return sum(np.prod([A[i, p[i]] for i in range(n)]) for p in itertools.permutations(range(n))) if n else 1.0


@pytest.mark.parametrize("n", range(0, 8))
def test_ryser_and_naive_vs_definition(n, rng):
    for _ in range(3):
        A = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        ref = perm_definition(A)
        assert abs(oracle.permanent(A, "ryser") - ref) <= 1e-12 * max(1, abs(ref))
        assert abs(oracle.permanent(A, "naive") - ref) <= 1e-12 * max(1, abs(ref))


def test_permanent_closed_forms(rng):
    for n in range(1, 13):
        assert abs(oracle.permanent(np.eye(n)) - 1) < 1e-14
        assert abs(oracle.permanent(np.ones((n, n))) - math.factorial(n)) <= 1e-12 * math.factorial(n)
        d = rng.normal(size=n) + 1j * rng.normal(size=n)
        assert abs(oracle.permanent(np.diag(d)) - np.prod(d)) < 1e-12 * max(1, abs(np.prod(d)))
    a, b, c, d = 1 + 2j, 3 - 1j, -0.5j, 2.0
    assert abs(oracle.permanent(np.array([[a, b], [c, d]])) - (a * d + b * c)) < 1e-14


def test_permanent_invariances(rng):
    n = 9
    A = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    p = oracle.permanent(A)
    assert abs(oracle.permanent(A.T) - p) < 1e-10 * abs(p)
    P = rng.permutation(n)
    Q = rng.permutation(n)
    assert abs(oracle.permanent(A[P][:, Q]) - p) < 1e-10 * abs(p)
    # multilinear in each row
    B = A.copy()
    B[3] *= 2.5
    assert abs(oracle.permanent(B) - 2.5 * p) < 1e-10 * abs(p)


def test_circuit_unitary_properties(rng):
    for M, D in [(2, 1), (6, 3), (7, 5), (16, 4)]:
        layers = li.clements_mesh(M, D, seed=M * 10 + D)
        U = oracle.circuit_unitary(M, layers)
        assert np.abs(U.conj().T @ U - np.eye(M)).max() < 1e-13
    assert np.abs(oracle.circuit_unitary(5, []) - np.eye(5)).max() == 0
    th, ph = 0.4, 2.2
    U = oracle.circuit_unitary(2, [[(0, 1, th, ph)]])
    want = np.array([[math.cos(th), -np.exp(-1j * ph) * math.sin(th)], [np.exp(1j * ph) * math.sin(th), math.cos(th)]])
    assert np.abs(U - want).max() < 1e-15
    # reversed port order is the conjugation by the swap
    Ur = oracle.circuit_unitary(2, [[(1, 0, th, ph)]])
    Psw = np.array([[0, 1], [1, 0]])
    assert np.abs(Ur - Psw @ want @ Psw).max() < 1e-15
    # concatenation: later layers multiply on the left
    A = li.random_nn_circuit(6, 3, rng)
    B = li.random_nn_circuit(6, 2, rng)
    UA, UB, UAB = (oracle.circuit_unitary(6, x) for x in (A, B, A + B))
    assert np.abs(UAB - UB @ UA).max() < 1e-13


def test_single_bs_amplitude_is_appendix_a(rng):
    """The permanent route and the Appendix-A route agree on one BS."""
    for _ in range(5):
        th, ph = rng.uniform(0, math.pi / 2), rng.uniform(0, 2 * math.pi)
        for n in range(0, 7):
            for x1 in range(n + 1):
                T = np.array([[y1, n - y1] for y1 in range(n + 1)])
                a = oracle.amplitudes_permanent(2, [[(0, 1, th, ph)]], [x1, n - x1], T)
                b = np.array([oracle.bs_element(th, ph, x1, n - x1, y1, n - y1) for y1 in range(n + 1)])
                assert np.abs(a - b).max() < 1e-13
