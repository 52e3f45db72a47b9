"""Pins for the oracle's photon-number-preserving phase gates (reading R19).

A gate on mode m after layer j multiplies a path by exp(i (a n + b n^2)), n = photons in
mode m after layer j.  Pinned to:
  * closed forms: gates on the input (j = 0) or on the output (j = D) see a fixed photon
    number, so they multiply the amplitude by exp(i (a S_m + b S_m^2)) / (.. T_m ..);
  * linear gates (b = 0) are phase shifters diag(e^{i a}) on mode m between layers j and
    j+1 of the single-particle unitary, so the amplitude equals the Ryser permanent of
    U_D..U_{j+1} P U_j..U_1;
  * Kerr gates (b != 0) anywhere: a state-vector evolution through the Fock space (a
    different algorithm from the path recursion), each BS applied with its two-mode
    Fock block and each gate as a diagonal phase.
"""
import cmath
import math
from collections import defaultdict

import numpy as np
import pytest

import lofp_inputs as li
import oracle


def phase(a, b, n):
    return cmath.exp(1j * (a * n + b * n * n))


def random_case(seed, M=5, D=4, N=3):
    rng = np.random.default_rng(seed)
    layers = li.random_nn_circuit(M, D, rng, fill=0.9, reverse_prob=0.2)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    return rng, layers, S


@pytest.mark.parametrize("seed", range(4))
def test_gates_on_input_and_output_closed_form(seed):
    rng, layers, S = random_case(seed)
    M, D = len(S), len(layers)
    T = li.all_outputs(M, int(S.sum()))
    base = oracle.path_sum(M, layers, S, T)
    m0, m1 = int(rng.integers(0, M)), int(rng.integers(0, M))
    a0, b0, a1, b1 = rng.uniform(-3, 3, size=4)
    got = oracle.path_sum(M, layers, S, T, gates=[(m0, 0, a0, b0), (m1, D, a1, b1)])
    want = base * phase(a0, b0, int(S[m0])) * np.array([phase(a1, b1, int(t[m1])) for t in T])
    assert np.abs(got - want).max() < 1e-14


def unitary_with_phase(M, layers, j, m, a):
    U1 = oracle.circuit_unitary(M, layers[:j])
    U2 = oracle.circuit_unitary(M, layers[j:])
    P = np.eye(M, dtype=complex)
    P[m, m] = cmath.exp(1j * a)
    return U2 @ P @ U1


def amp_ryser(U, S, T):
    rows = [i for i in range(len(T)) for _ in range(int(T[i]))]
    cols = [j for j in range(len(S)) for _ in range(int(S[j]))]
    A = U[np.ix_(rows, cols)]
    norm = math.sqrt(math.prod(math.factorial(int(x)) for x in S) * math.prod(math.factorial(int(x)) for x in T))
    return oracle.permanent(A) / norm


@pytest.mark.parametrize("seed", range(6))
def test_linear_gate_is_a_phase_shifter(seed):
    rng, layers, S = random_case(100 + seed, M=6, D=5, N=4)
    M, D = len(S), len(layers)
    j, m, a = int(rng.integers(1, D)), int(rng.integers(0, M)), float(rng.uniform(-3, 3))
    U = unitary_with_phase(M, layers, j, m, a)
    T = li.all_outputs(M, int(S.sum()))
    got = oracle.path_sum(M, layers, S, T, gates=[(m, j, a, 0.0)])
    want = np.array([amp_ryser(U, S, t) for t in T])
    assert np.abs(got - want).max() < 1e-13


def evolve(M, layers, S, gates):
    """Fock-space state vector: {occupation tuple: amplitude}."""
    state = {tuple(int(x) for x in S): 1.0 + 0j}

    def apply_gates(state, j):
        for (m, jj, a, b) in gates:
            if jj == j:
                state = {k: v * phase(a, b, k[m]) for k, v in state.items()}
        return state

    state = apply_gates(state, 0)
    for j, layer in enumerate(layers, start=1):
        for (ma, mb, th, ph) in layer:
            new = defaultdict(complex)
            for k, v in state.items():
                x1, x2 = k[ma], k[mb]
                for y1 in range(x1 + x2 + 1):
                    e = oracle.bs_element(th, ph, x1, x2, y1, x1 + x2 - y1)
                    kk = list(k)
                    kk[ma], kk[mb] = y1, x1 + x2 - y1
                    new[tuple(kk)] += v * e
            state = dict(new)
        state = apply_gates(state, j)
    return state


@pytest.mark.parametrize("seed", range(6))
def test_kerr_gates_against_state_vector(seed):
    rng, layers, S = random_case(200 + seed, M=5, D=5, N=4)
    M, D = len(S), len(layers)
    gates = [(int(rng.integers(0, M)), int(rng.integers(0, D + 1)), float(rng.uniform(-2, 2)),
              float(rng.uniform(-2, 2))) for _ in range(5)]
    T = li.all_outputs(M, int(S.sum()))
    got = oracle.path_sum(M, layers, S, T, gates=gates)
    sv = evolve(M, layers, S, gates)
    want = np.array([sv.get(tuple(int(x) for x in t), 0.0) for t in T])
    assert np.abs(got - want).max() < 1e-13
    assert abs(np.sum(np.abs(got) ** 2) - 1.0) < 1e-13  # gates are unitary
