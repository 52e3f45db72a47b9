"""GPU parity of the strip tensor contraction (NEXT-1; lofp_amplitudes_contract).

The contraction evaluates eq. (1) without forming path products, so it reaches outputs no
enumerator can: configs[3] as literally drawn (BASELINE.json: 2048 outputs of up to 1.5e16
paths each) is checked output by output against the Ryser permanent (n = 12).  Elsewhere it
is checked against the oracle path sum and against the GPU path-sum engine.
Tolerance (BASELINE.json north_star): |a - a_ref| <= 1e-12 + 1e-9 |a_ref|.
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


def contract(lofp, M, layers, S, T, gates=()):
    circ = lofp.Circuit(M, layers, gates)
    Td = torch.from_numpy(np.ascontiguousarray(T, dtype=np.int32)).cuda()
    counts = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    a = circ.contract(S, Td, counts=counts)
    torch.cuda.synchronize()
    return a.cpu().numpy(), counts.cpu().numpy().astype(np.uint64), circ.stats()


def paths(lofp, M, layers, S, T, gates=()):
    circ = lofp.Circuit(M, layers, gates)
    a = circ.amplitudes(S, torch.from_numpy(np.ascontiguousarray(T, dtype=np.int32)).cuda())
    torch.cuda.synchronize()
    return a.cpu().numpy()


def load(idx):
    return np.load(os.path.join(ROOT, "data", f"cfg{idx}.npz"))


def test_config0_and_unitarity(lofp):
    c = li.config(0)
    T = c.draw_outputs()
    got, cnt, st = contract(lofp, c.M, c.layers, c.S, T)
    ref, leaves = oracle.path_sum(c.M, c.layers, c.S, T, return_leaves=True)
    assert tol_ok(got, ref)[0]
    assert np.array_equal(cnt, leaves)
    assert abs(np.sum(np.abs(got) ** 2) - 1) < 1e-12
    assert st["mode"] == 1 and st["terms"] > 0


@pytest.mark.parametrize("seed", range(12))
def test_random_circuits_with_gates(lofp, seed):
    rng = np.random.default_rng(5100 + seed)
    M = int(rng.integers(1, 10))
    D = int(rng.integers(0, 8))
    N = int(rng.integers(0, 6))
    layers = li.random_nn_circuit(M, D, rng, fill=float(rng.uniform(0.4, 1.0)), reverse_prob=0.4)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    gates = [(int(rng.integers(0, M)), int(rng.integers(0, D + 1)), float(rng.uniform(-3, 3)),
              float(rng.uniform(-1, 1))) for _ in range(int(rng.integers(0, 4)))]
    T = li.all_outputs(M, N)
    if len(T) > 300:
        T = T[rng.choice(len(T), 300, replace=False)]
    T = np.concatenate([T, np.clip(T[:3] + 1, 0, None)])
    got, cnt, _ = contract(lofp, M, layers, S, T, gates)
    ref, leaves = oracle.path_sum(M, layers, S, T, return_leaves=True, gates=gates)
    ok, err = tol_ok(got, ref)
    assert ok, err
    assert np.array_equal(cnt, leaves)


def test_config1_literal(lofp):
    c = li.config(1)
    d = load(1)
    T = d["T_literal"].astype(np.int32)
    got, cnt, _ = contract(lofp, c.M, c.layers, c.S, T)
    assert np.array_equal(cnt, d["P_literal"])
    assert tol_ok(got, oracle.path_sum(c.M, c.layers, c.S, T))[0]


@pytest.mark.parametrize("idx", [2, 3, 4])
def test_conditioned_batches_match_path_engine(lofp, idx):
    """Two GPU algorithms, one sum: the contraction against the path-sum engine on the full
    conditioned batch, and against Ryser on a sample."""
    c = li.config(idx)
    d = load(idx)
    T = d["T_cond"].astype(np.int32)
    got, cnt, st = contract(lofp, c.M, c.layers, c.S, T)
    assert np.array_equal(cnt, d["P_cond"])
    assert st["unsupported"] == 0
    assert tol_ok(got, paths(lofp, c.M, c.layers, c.S, T))[0]
    pick = np.random.default_rng(idx).choice(len(T), 64, replace=False)
    assert tol_ok(got[pick], oracle.amplitudes_permanent(c.M, c.layers, c.S, T[pick]))[0]


def test_config3_literal_batch_all_outputs_vs_ryser(lofp):
    """configs[3] exactly as BASELINE.json draws it: 2048 outputs, up to 1.5e16 paths each
    (2.5e18 in total) -- every amplitude against the Ryser permanent (n = 12)."""
    c = li.config(3)
    d = load(3)
    T = d["T_literal"].astype(np.int32)
    got, cnt, st = contract(lofp, c.M, c.layers, c.S, T)
    assert np.array_equal(cnt, d["P_literal"])
    assert st["unsupported"] == 0 and st["check_errors"] == 0
    ref = oracle.amplitudes_permanent(c.M, c.layers, c.S, T)
    ok, err = tol_ok(got, ref)
    assert ok, err


def test_config2_literal_batch(lofp):
    c = li.config(2)
    d = load(2)
    T = d["T_literal"].astype(np.int32)
    got, cnt, _ = contract(lofp, c.M, c.layers, c.S, T)
    assert np.array_equal(cnt, d["P_literal"])
    reach = d["P_literal"] > 0
    assert (got[~reach] == 0).all()
    ref = oracle.amplitudes_permanent(c.M, c.layers, c.S, T[reach])
    assert tol_ok(got[reach], ref)[0]


@pytest.mark.parametrize("D", [3, 4])
def test_density_workload_all_densities(lofp, D):
    """P:318 at every density k = 1..10 (10..100 photons in 10 modes): the contraction and
    the path-sum engine agree (D = 4, k = 10 is 2.3e11 paths); the oracle at k <= 3."""
    M = 10
    layers = li.clements_mesh(M, D, seed=318 + D)
    for k in range(1, 11):
        S = np.full(M, k, dtype=np.int32)
        a, cnt, st = contract(lofp, M, layers, S, S[None, :])
        b = paths(lofp, M, layers, S, S[None, :])
        assert np.isfinite(a).all() and st["unsupported"] == 0
        ok, err = tol_ok(a, b)
        assert ok, (k, err)
        if k <= 3:
            assert tol_ok(a, oracle.path_sum(M, layers, S, S[None, :]))[0]


@pytest.mark.parametrize("method", ["contract", "paths"])
def test_distribution_paper_protocol(lofp, method):
    """NEXT-2: all output amplitudes of one input in one call.  The paper's §III.A
    protocol: its four 6-mode inputs at depths 3..6, probabilities of every
    output summing to 1 and their total variation distance to Ryser's far below 1e-13."""
    for case, (S, D) in enumerate(li.paper_correctness_inputs()):
        S = np.array(S, dtype=np.int32)
        layers = li.clements_mesh(6, D, seed=300 + case)
        circ = lofp.Circuit(6, layers)
        T, a = circ.distribution(S, method=method)
        torch.cuda.synchronize()
        T = T.cpu().numpy()
        a = a.cpu().numpy()
        assert np.array_equal(T, li.all_outputs(6, int(S.sum())))  # every pattern, fixed order
        p = np.abs(a) ** 2
        assert abs(p.sum() - 1.0) < 1e-12
        q = np.abs(oracle.amplitudes_permanent(6, layers, S, T)) ** 2
        assert oracle.tvd(p, q) < 1e-13


def test_distribution_config1_unitarity(lofp):
    """configs[1]'s circuit and input: all C(23, 8) = 490,314 outputs in one call; the
    probabilities sum to 1 (unitarity) and a sample matches the oracle."""
    c = li.config(1)
    circ = lofp.Circuit(c.M, c.layers)
    T, a = circ.distribution(c.S)
    torch.cuda.synchronize()
    T = T.cpu().numpy()
    a = a.cpu().numpy()
    assert len(T) == 490314
    assert abs(np.sum(np.abs(a) ** 2) - 1.0) < 1e-11
    pick = np.random.default_rng(1).choice(len(T), 200, replace=False)
    assert tol_ok(a[pick], oracle.path_sum(c.M, c.layers, c.S, T[pick]))[0]


def test_warp_kernel_matches_block_kernel(lofp, monkeypatch):
    """The warp-per-output contraction (lofp_contract.cu) and the block-per-output kernel
    (forced by LOFP_CONTRACT_BLOCK) compute the same amplitudes and path counts on configs[3]
    as literally drawn; the warp kernel defers none of them."""
    c = li.config(3)
    d = load(3)
    T = d["T_literal"][:512].astype(np.int32)
    a_w, cnt_w, st_w = contract(lofp, c.M, c.layers, c.S, T)
    assert st_w["contract_deferred"] == 0 and st_w["check_errors"] == 0
    monkeypatch.setenv("LOFP_CONTRACT_BLOCK", "1")
    a_b, cnt_b, st_b = contract(lofp, c.M, c.layers, c.S, T)
    assert np.array_equal(cnt_w, cnt_b) and np.array_equal(cnt_w, d["P_literal"][:512])
    ok, err = tol_ok(a_w, a_b)
    assert ok, err


def test_warp_kernel_deterministic(lofp):
    """Each output is summed by one warp in a fixed order: repeated calls are bitwise equal."""
    c = li.config(3)
    T = load(3)["T_literal"][:256].astype(np.int32)
    circ = lofp.Circuit(c.M, c.layers)
    Td = torch.from_numpy(T).cuda()
    a = circ.contract(c.S, Td).cpu().numpy()
    for _ in range(3):
        assert np.array_equal(circ.contract(c.S, Td).cpu().numpy(), a)


@pytest.mark.parametrize("N", [1, 2])
def test_deep_circuit_defers_to_block_kernel(lofp, N):
    """16 layers put 9 segments in a column (more than the warp kernel's packed 8): those
    outputs are deferred in the same call to the block kernel (N = 1) or, past its column
    limits, to the generic engine (N = 2); parity with the oracle either way."""
    M, D = 4, 16
    layers = li.clements_mesh(M, D, seed=1616)
    S = np.array([1, 1, 0, 0][:M], dtype=np.int32) if N == 2 else np.array([0, 1, 0, 0], dtype=np.int32)
    T = li.all_outputs(M, N)
    got, cnt, st = contract(lofp, M, layers, S, T)
    assert st["contract_deferred"] > 0 and st["unsupported"] == 0
    ref, leaves = oracle.path_sum(M, layers, S, T, return_leaves=True)
    assert tol_ok(got, ref)[0]
    assert np.array_equal(cnt, leaves)
    assert abs(np.sum(np.abs(got) ** 2) - 1) < 1e-12



def test_small_scratch(lofp, monkeypatch):
    """The smallest per-block scratch the library accepts (LOFP_SLAB_MB below 2 is raised to
    2): the warp kernel's slices shrink with it; every output is still evaluated."""
    monkeypatch.setenv("LOFP_SLAB_MB", "1")
    c = li.config(1)
    d = load(1)
    T = np.tile(d["T_literal"].astype(np.int32), (3, 1))
    got, cnt, st = contract(lofp, c.M, c.layers, c.S, T)
    assert st["unsupported"] == 0 and st["check_errors"] == 0
    assert np.array_equal(cnt, np.tile(d["P_literal"], 3))
    monkeypatch.delenv("LOFP_SLAB_MB")
    ref, _, _ = contract(lofp, c.M, c.layers, c.S, T)
    assert tol_ok(got, ref)[0]


@pytest.mark.parametrize("counts", [False, True])
def test_eight_lane_groups_match_full_warps(lofp, monkeypatch, counts):
    """Small circuits in large batches run with 8 lanes per output (four outputs per warp);
    forced on and off (LOFP_CONTRACT_GROUP) on configs[1]'s literal batch tiled to 40960
    outputs, and on random small circuits with gates: same amplitudes and path counts."""
    c = li.config(1)
    d = load(1)
    T = np.tile(d["T_literal"].astype(np.int32), (40, 1))
    res = {}
    for grp in ("8", "32"):
        monkeypatch.setenv("LOFP_CONTRACT_GROUP", grp)
        circ = lofp.Circuit(c.M, c.layers)
        Td = torch.from_numpy(T).cuda()
        cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda") if counts else None
        a = circ.contract(c.S, Td, counts=cnt).cpu().numpy()
        res[grp] = (a, None if cnt is None else cnt.cpu().numpy().astype(np.uint64))
    assert tol_ok(res["8"][0], res["32"][0])[0]
    assert tol_ok(res["8"][0][:1024], oracle.path_sum(c.M, c.layers, c.S, T[:1024]))[0]
    if counts:
        assert np.array_equal(res["8"][1], res["32"][1])
        assert np.array_equal(res["8"][1][:1024], d["P_literal"])
    rng = np.random.default_rng(808)
    for _ in range(6):
        M = int(rng.integers(2, 12))
        D = int(rng.integers(1, 7))
        N = int(rng.integers(1, 5))
        layers = li.random_nn_circuit(M, D, rng, fill=0.8, reverse_prob=0.3)
        S = np.zeros(M, dtype=np.int32)
        for m in rng.integers(0, M, size=N):
            S[m] += 1
        gates = [(int(rng.integers(0, M)), int(rng.integers(0, D + 1)), float(rng.uniform(-3, 3)),
                  float(rng.uniform(-1, 1))) for _ in range(int(rng.integers(0, 3)))]
        Tr = li.all_outputs(M, N)
        monkeypatch.setenv("LOFP_CONTRACT_GROUP", "8")
        got, cnt, _ = contract(lofp, M, layers, S, Tr, gates)
        ref, leaves = oracle.path_sum(M, layers, S, Tr, return_leaves=True, gates=gates)
        assert tol_ok(got, ref)[0]
        assert np.array_equal(cnt, leaves)


@pytest.mark.parametrize("counts", [False, True])
def test_entry_schedule_does_not_change_results(lofp, monkeypatch, counts):
    """The warp kernel takes a cut's entries longest row first (a counting sort by row length);
    with LOFP_CONTRACT_NOSORT it takes them in storage order.  Every entry's sum is formed in
    the same order either way: bitwise equal amplitudes and equal path counts on configs[3] as
    literally drawn (levels of several rounds) and on a high-density output (k = 6)."""
    c = li.config(3)
    d = load(3)
    T = d["T_literal"][:384].astype(np.int32)
    layers318 = li.clements_mesh(10, 4, 318 + 4)
    S318 = np.full(10, 6, dtype=np.int32)
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("LOFP_CONTRACT_NOSORT", flag)
        circ = lofp.Circuit(c.M, c.layers)
        Td = torch.from_numpy(T).cuda()
        cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda") if counts else None
        a = circ.contract(c.S, Td, counts=cnt).cpu().numpy()
        circ2 = lofp.Circuit(10, layers318)
        b = circ2.contract(S318, torch.from_numpy(S318[None, :].copy()).cuda()).cpu().numpy()
        res[flag] = (a, None if cnt is None else cnt.cpu().numpy().astype(np.uint64), b)
    assert np.array_equal(res["0"][0], res["1"][0]) and np.array_equal(res["0"][2], res["1"][2])
    if counts:
        assert np.array_equal(res["0"][1], res["1"][1])
        assert np.array_equal(res["0"][1], d["P_literal"][:384])
