"""Pins for the oracle's Appendix-A element at high photon numbers (P:354-408, P:318's
density workload reaches 80+ photons through one BS; reading R18).

The oracle sums Appendix A's alternating t-sum in __float128.  These tests pin it, up
to the library's 120-photon limit, to things it does not compute that way:

  * the single-mode-input row in closed form: a1^dag -> c b1^dag + e^{i phi} s b2^dag
    (eq. bs_matrix), so <y1, n-y1|BS|n, 0> = sqrt(C(n, y1)) c^y1 (e^{i phi} s)^(n-y1)
    (binomial expansion), and the mirrored row for |0, n>;
  * unitarity of the whole (n+1)x(n+1) block (the Fock representation of a unitary);
  * an independent algorithm: the four-term creation-operator recurrence
        n d_n(x, y) = sum_{i,k} sqrt(x_i y_k) u_ki d_{n-1}(x - e_i, y - e_k)
    (from sqrt(x_i) <y|U|x> = sum_k u_ki sqrt(y_k) <y - e_k|U|x - e_i>), run in float64,
    which is numerically stable (no cancellation), with the phase e^{i phi (x1 - y1)}.
"""
import math

import numpy as np
import pytest

import oracle


def recurrence_block(theta, phi, n):
    """<y1, n-y1| BS |x1, n-x1> for all x1, y1 by the four-term recurrence (test-side)."""
    c, s = math.cos(theta), math.sin(theta)
    u = np.array([[c, -s], [s, c]])  # the real rotation; the phase is restored below
    d = np.ones((1, 1))
    for m in range(1, n + 1):
        nd = np.zeros((m + 1, m + 1))
        x1 = np.arange(m + 1)[:, None]
        y1 = np.arange(m + 1)[None, :]
        x = (x1, m - x1)
        y = (y1, m - y1)
        for i in range(2):
            for k in range(2):
                px1 = x1 - (1 if i == 0 else 0)
                py1 = y1 - (1 if k == 0 else 0)
                ok = (x[i] > 0) & (y[k] > 0) & (px1 >= 0) & (px1 <= m - 1) & (py1 >= 0) & (py1 <= m - 1)
                val = np.where(ok, d[np.clip(px1, 0, m - 1), np.clip(py1, 0, m - 1)], 0.0)
                nd += np.sqrt(np.where(ok, x[i] * y[k], 0)) * u[k, i] * val
        d = nd / m
    x1 = np.arange(n + 1)[:, None]
    y1 = np.arange(n + 1)[None, :]
    return d * np.exp(1j * phi * (x1 - y1))


def oracle_block(theta, phi, n):
    B = np.zeros((n + 1, n + 1), dtype=complex)
    for x1 in range(n + 1):
        for y1 in range(n + 1):
            B[x1, y1] = oracle.bs_element(theta, phi, x1, n - x1, y1, n - y1)
    return B


@pytest.mark.parametrize("n", [30, 60, 90, 120])
def test_single_mode_input_closed_form(n):
    rng = np.random.default_rng(n)
    for _ in range(3):
        th, ph = rng.uniform(0, math.pi / 2), rng.uniform(0, 2 * math.pi)
        c, s = math.cos(th), math.sin(th)
        for y1 in range(0, n + 1, max(1, n // 12)):
            binom = math.comb(n, y1)
            # |n, 0> -> sum_y1 sqrt(C(n,y1)) c^y1 (e^{i phi} s)^(n-y1) |y1, n-y1>
            want = math.sqrt(binom) * c ** y1 * (np.exp(1j * ph) * s) ** (n - y1)
            got = oracle.bs_element(th, ph, n, 0, y1, n - y1)
            assert abs(got - want) <= 1e-14 + 1e-12 * abs(want), (n, y1)
            # |0, n> -> sum_y1 sqrt(C(n,y1)) (-e^{-i phi} s)^y1 c^(n-y1) |y1, n-y1>
            want = math.sqrt(binom) * (-np.exp(-1j * ph) * s) ** y1 * c ** (n - y1)
            got = oracle.bs_element(th, ph, 0, n, y1, n - y1)
            assert abs(got - want) <= 1e-14 + 1e-12 * abs(want), (n, y1)


@pytest.mark.parametrize("n", [40, 80, 120])
def test_block_unitary_and_recurrence(n):
    rng = np.random.default_rng(1000 + n)
    th, ph = rng.uniform(0, math.pi / 2), rng.uniform(0, 2 * math.pi)
    B = oracle_block(th, ph, n)
    assert np.isfinite(B).all()
    # rows x1 (inputs), columns y1 (outputs): B^T is the n-photon block of the unitary
    assert np.abs(B.conj() @ B.T - np.eye(n + 1)).max() < 1e-13
    R = recurrence_block(th, ph, n)
    assert np.abs(B - R).max() < 1e-13


def test_recurrence_helper_matches_low_n_definition():
    """The test-side recurrence itself agrees with the oracle where the t-sum is exact."""
    th, ph = 0.61, 2.3
    for n in range(0, 9):
        assert np.abs(recurrence_block(th, ph, n) - oracle_block(th, ph, n)).max() < 1e-15


def test_limit_is_enforced():
    assert math.isnan(oracle.bs_element(0.3, 0.1, 121, 0, 121, 0).real)


@pytest.mark.parametrize("D,k", [(3, 1), (3, 2), (4, 1), (4, 2)])
def test_density_workload_pathsum_vs_ryser(D, k):
    """P:318's density workload (10 modes, depth 3/4, S = T = (k,...,k)) at the densities
    where Ryser (n = 10k photons, 2^n terms) is still cheap."""
    import lofp_inputs as li
    M = 10
    layers = li.clements_mesh(M, D, seed=318 + D)
    S = np.full(M, k, dtype=np.int32)
    a, leaves = oracle.path_sum(M, layers, S, S[None, :], return_leaves=True)
    r = oracle.amplitudes_permanent(M, layers, S, S[None, :])
    assert abs(a[0] - r[0]) <= 1e-13 + 1e-10 * abs(r[0])
    assert int(leaves[0]) == oracle.count_paths(M, layers, S, S[None, :])[0]
