"""GPU parity for circuits with non-local pairs (NEXT-4; "non-local connections").

The column model carries a long BS's photon numbers through the columns it spans (DESIGN.md
R21), so the path-sum engine, the contraction and the distribution mode all accept such
circuits.  Reference: the oracle path sum with the paper's cone bounds (pinned to
Ryser and to the unpruned sum on non-local circuits in test_oracle_pathsum.py), whose leaf
count is the exact number of valid paths.
"""
import os

import numpy as np
import pytest

import lofp_inputs as li
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lofp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2510_26408_b200 as pkg
    return pkg


def tol_ok(got, ref):
    err = np.abs(np.asarray(got) - np.asarray(ref))
    return bool((err <= 1e-12 + 1e-9 * np.abs(ref)).all()), float(err.max()) if err.size else 0.0


def case(seed, Mr=(3, 9), Dr=(1, 6), Nr=(1, 6)):
    rng = np.random.default_rng(6100 + seed)
    M = int(rng.integers(*Mr))
    D = int(rng.integers(*Dr))
    N = int(rng.integers(*Nr))
    layers = li.random_nonlocal_circuit(M, D, rng, fill=float(rng.uniform(0.5, 1.0)))
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    T = li.all_outputs(M, N)
    if len(T) > 250:
        T = T[rng.choice(len(T), 250, replace=False)]
    return rng, M, layers, S, T


@pytest.mark.parametrize("seed", range(16))
def test_nonlocal_path_sum_and_contraction(lofp, seed):
    rng, M, layers, S, T = case(seed)
    ref, leaves = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_CONE, return_leaves=True)
    circ = lofp.Circuit(M, layers)
    Td = torch.from_numpy(T).cuda()
    cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    a = circ.amplitudes(S, Td, counts=cnt).cpu().numpy()
    st = circ.stats()
    assert st["check_errors"] == 0 and st["unsupported"] == 0
    ok, err = tol_ok(a, ref)
    assert ok, err
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), leaves)
    cnt2 = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    b = circ.contract(S, Td, counts=cnt2).cpu().numpy()
    ok, err = tol_ok(b, ref)
    assert ok, err
    assert np.array_equal(cnt2.cpu().numpy().astype(np.uint64), leaves)


@pytest.mark.parametrize("seed", range(4))
def test_nonlocal_with_gates_and_distribution(lofp, seed):
    """Phase gates on a non-local circuit, and the full output distribution (sum p = 1,
    TVD to Ryser)."""
    rng, M, layers, S, T = case(100 + seed, Mr=(4, 7), Dr=(2, 5), Nr=(2, 5))
    D = len(layers)
    gates = [(int(rng.integers(0, M)), int(rng.integers(0, D + 1)), float(rng.uniform(-2, 2)),
              float(rng.uniform(-1, 1))) for _ in range(3)]
    circ = lofp.Circuit(M, layers, gates)
    a = circ.amplitudes(S, torch.from_numpy(T).cuda()).cpu().numpy()
    ref = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_CONE, gates=gates)
    assert tol_ok(a, ref)[0]
    plain = lofp.Circuit(M, layers)
    To, amp = plain.distribution(S)
    torch.cuda.synchronize()
    To = To.cpu().numpy()
    p = np.abs(amp.cpu().numpy()) ** 2
    assert abs(p.sum() - 1) < 1e-12
    q = np.abs(oracle.amplitudes_permanent(M, layers, S, To)) ** 2
    assert oracle.tvd(p, q) < 1e-12


def test_long_range_mesh(lofp):
    """A 12-mode brickwork mesh with long-range couplers added in every other layer (mode i
    to mode i+5): a wide, non-local circuit; values against Ryser, counts against the oracle."""
    M, D = 12, 4
    layers = li.clements_mesh(M, D, seed=71)
    rng = np.random.default_rng(71)
    for l in (1, 3):  # replace two NN pairs of the layer by one long pair
        layer = [bs for bs in layers[l] if bs[0] not in (3, 4, 7, 8) and bs[1] not in (3, 4, 7, 8)]
        layer.append((3, 8, float(rng.uniform(0, 1.5)), float(rng.uniform(0, 6))))
        layers[l] = layer
    S = np.zeros(M, dtype=np.int32)
    S[[0, 2, 4, 6, 8, 10]] = 1
    T = li.all_outputs(M, 6)
    T = T[np.random.default_rng(5).choice(len(T), 300, replace=False)]
    circ = lofp.Circuit(M, layers)
    cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    a = circ.amplitudes(S, torch.from_numpy(T).cuda(), counts=cnt).cpu().numpy()
    ref = oracle.amplitudes_permanent(M, layers, S, T)
    ok, err = tol_ok(a, ref)
    assert ok, err
    _, leaves = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_CONE, return_leaves=True)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), leaves)


@pytest.mark.parametrize("seed", range(6))
def test_generic_engine_forced(lofp, seed, monkeypatch):
    """The generic engine (the paper's layer-major recursion with its cone bounds, P:100,
    P:164) on its own: every output routed to it, local and non-local circuits, with gates;
    values and valid-path counts against the oracle."""
    monkeypatch.setenv("LOFP_FORCE_GENERIC", "1")
    rng, M, layers, S, T = case(200 + seed)
    if seed % 2:
        layers = li.random_nn_circuit(M, len(layers), rng, fill=0.8, reverse_prob=0.3)
    D = len(layers)
    gates = [(int(rng.integers(0, M)), int(rng.integers(0, D + 1)), float(rng.uniform(-2, 2)),
              float(rng.uniform(-1, 1))) for _ in range(2)]
    circ = lofp.Circuit(M, layers, gates)
    cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    a = circ.amplitudes(S, torch.from_numpy(T).cuda(), counts=cnt).cpu().numpy()
    st = circ.stats()
    ref, leaves = oracle.path_sum(M, layers, S, T, prune=oracle.PRUNE_CONE, return_leaves=True, gates=gates)
    ok, err = tol_ok(a, ref)
    assert ok, err
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), leaves)
    assert st["generic"] == len(T) and st["unsupported"] == 0  # (every row has the right photon number)
