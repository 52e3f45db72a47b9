"""Pins for oracle_bs_element (Appendix A, reading R1).

The oracle evaluates the closed t-sum; these tests pin it to things it does not
compute that way: the permanent of the expanded matrix by brute force over
permutations, the Hong-Ou-Mandel closed forms (golden fixture), the
unitarity of the multi-photon BS, and the theta = 0 / pi/2 special cases.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def bs_u(theta, phi):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -np.exp(-1j * phi) * s], [np.exp(1j * phi) * s, c]])


def expanded_permanent_amp(theta, phi, x1, x2, y1, y2):
    """y1 rows (U11 x1 times, U12 x2 times), y2 rows (U21 x1 times, U22 x2 times);
    permanent by the definition / sqrt(x1!x2!y1!y2!)."""
    u = bs_u(theta, phi)
    n = x1 + x2
    rows = [[u[0, 0]] * x1 + [u[0, 1]] * x2] * y1 + [[u[1, 0]] * x1 + [u[1, 1]] * x2] * y2
    A = np.array(rows, dtype=complex).reshape(n, n)
    per = sum(np.prod([A[i, p[i]] for i in range(n)]) for p in itertools.permutations(range(n))) if n else 1.0
    return per / math.sqrt(math.factorial(x1) * math.factorial(x2) * math.factorial(y1) * math.factorial(y2))


def test_hom_golden():
    g = json.load(open(os.path.join(GOLDEN, "hom.json")))
    for case in g["cases"]:
        a = oracle.bs_element(g["theta"], g["phi"], *case["x"], *case["y"])
        assert abs(a - complex(case["re"], case["im"])) <= g["tolerance"]


@pytest.mark.parametrize("seed", range(5))
def test_two_photon_closed_forms(seed):
    rng = np.random.default_rng(seed)
    th, ph = rng.uniform(0, math.pi / 2), rng.uniform(0, 2 * math.pi)
    c, s = math.cos(th), math.sin(th)
    assert abs(oracle.bs_element(th, ph, 1, 1, 1, 1) - math.cos(2 * th)) < 1e-15
    assert abs(oracle.bs_element(th, ph, 1, 1, 2, 0) - (-math.sqrt(2) * c * s * np.exp(-1j * ph))) < 1e-15
    assert abs(oracle.bs_element(th, ph, 1, 1, 0, 2) - (math.sqrt(2) * c * s * np.exp(1j * ph))) < 1e-15
    # single photon: the 2x2 matrix itself (rows = outputs, columns = inputs)
    u = bs_u(th, ph)
    assert abs(oracle.bs_element(th, ph, 1, 0, 1, 0) - u[0, 0]) < 1e-15
    assert abs(oracle.bs_element(th, ph, 0, 1, 1, 0) - u[0, 1]) < 1e-15
    assert abs(oracle.bs_element(th, ph, 1, 0, 0, 1) - u[1, 0]) < 1e-15
    assert abs(oracle.bs_element(th, ph, 0, 1, 0, 1) - u[1, 1]) < 1e-15


def test_against_expanded_permanent():
    rng = np.random.default_rng(7)
    angles = [(0.0, 0.0), (math.pi / 2, 0.3), (math.pi / 4, 0.0)] + [
        (rng.uniform(0, math.pi / 2), rng.uniform(0, 2 * math.pi)) for _ in range(20)]
    worst = 0.0
    for th, ph in angles:
        for n in range(0, 7):
            for x1 in range(n + 1):
                for y1 in range(n + 1):
                    a = oracle.bs_element(th, ph, x1, n - x1, y1, n - y1)
                    b = expanded_permanent_amp(th, ph, x1, n - x1, y1, n - y1)
                    worst = max(worst, abs(a - b))
    assert worst < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_multiphoton_unitarity(seed):
    """The N-photon BS is unitary: its columns (fixed input split) are orthonormal."""
    rng = np.random.default_rng(100 + seed)
    th, ph = rng.uniform(0, math.pi / 2), rng.uniform(0, 2 * math.pi)
    for n in range(0, 11):
        E = np.array([[oracle.bs_element(th, ph, x1, n - x1, y1, n - y1) for x1 in range(n + 1)]
                      for y1 in range(n + 1)])
        assert np.abs(E.conj().T @ E - np.eye(n + 1)).max() < 1e-12


def test_special_angles():
    for n in range(0, 8):
        for x1 in range(n + 1):
            x2 = n - x1
            for y1 in range(n + 1):
                y2 = n - y1
                ph = 0.9
                # theta = 0: identity
                assert abs(oracle.bs_element(0.0, ph, x1, x2, y1, y2) - (1.0 if y1 == x1 else 0.0)) < 1e-15
                # theta = pi/2: photons swap ports, amplitude U12^x2 U21^x1
                want = ((-np.exp(-1j * ph)) ** x2 * np.exp(1j * ph) ** x1) if y1 == x2 else 0.0
                assert abs(oracle.bs_element(math.pi / 2, ph, x1, x2, y1, y2) - want) < 1e-12


def test_phase_factorisation_and_conservation():
    rng = np.random.default_rng(3)
    for _ in range(10):
        th, ph = rng.uniform(0, math.pi / 2), rng.uniform(0, 2 * math.pi)
        for n in range(6):
            for x1 in range(n + 1):
                for y1 in range(n + 1):
                    a = oracle.bs_element(th, ph, x1, n - x1, y1, n - y1)
                    # BS = P(phi) R(theta) P(-phi): the element is e^{i phi (x1 - y1)} times a real number
                    assert abs((a * np.exp(-1j * ph * (x1 - y1))).imag) < 1e-14
                    # |element| does not depend on phi
                    assert abs(abs(a) - abs(oracle.bs_element(th, 0.0, x1, n - x1, y1, n - y1))) < 1e-14
    assert oracle.bs_element(0.3, 0.2, 1, 1, 1, 0) == 0  # photon number not conserved


def test_printed_factorial_fails_unitarity():
    """Reading R1: the factor (y1-x2+t)! printed at P:406 cannot be right — with it the
    single-BS map is not unitary, with (x2-y1+t)! it is (test_multiphoton_unitarity)."""
    th, ph = 0.61, 1.3
    u = bs_u(th, ph)

    def printed(x1, x2, y1, y2):
        tot = 0
        for t in range(max(0, y1 - x2, x1 - y2), min(x1, y1) + 1):
            if y1 - x2 + t < 0:
                return float("nan")
            tot += (math.factorial(y1) * math.factorial(x1) / (math.factorial(t) * math.factorial(y1 - t))
                    * math.factorial(y2) * math.factorial(x2)
                    / (math.factorial(x1 - t) * math.factorial(y1 - x2 + t))
                    * u[0, 0] ** t * u[0, 1] ** (y1 - t) * u[1, 0] ** (x1 - t) * u[1, 1] ** (x2 - y1 + t))
        return tot / math.sqrt(math.factorial(x1) * math.factorial(x2) * math.factorial(y1) * math.factorial(y2))

    n = 4
    col = [printed(1, 3, y1, n - y1) for y1 in range(n + 1)]
    assert not abs(sum(abs(c) ** 2 for c in col) - 1.0) < 1e-6
