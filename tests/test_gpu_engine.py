"""GPU tests of the column-split engine beyond the BASELINE configs: high photon density
(Appendix-A elements up to the 120-photon limit, P:318's density workload), phase gates
(P:338), stream ordering and CUDA-graph capture (the call never synchronises the host),
bitwise determinism, and the engine's internal splitting paths (units, sub-splits).

Tolerance (BASELINE.json north_star): |a - a_ref| <= 1e-12 + 1e-9 |a_ref| in fp64.
"""
import math
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


def run(lofp, M, layers, S, T, gates=()):
    circ = lofp.Circuit(M, layers, gates)
    Td = torch.from_numpy(np.ascontiguousarray(T, dtype=np.int32)).cuda()
    counts = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    a = circ.amplitudes(S, Td, counts=counts)
    torch.cuda.synchronize()
    return a.cpu().numpy(), counts.cpu().numpy().astype(np.uint64), circ.stats()


@pytest.mark.parametrize("n", [1, 10, 30, 60, 90, 120])
def test_single_bs_high_photon_numbers(lofp, n):
    """One BS, n photons split over its two inputs: every output against the oracle's
    __float128 Appendix-A element (reading R18); no inf/NaN anywhere up to the limit."""
    rng = np.random.default_rng(n)
    for _ in range(3):
        th, ph = float(rng.uniform(0, math.pi / 2)), float(rng.uniform(0, 2 * math.pi))
        x1 = int(rng.integers(0, n + 1))
        S = np.array([x1, n - x1], dtype=np.int32)
        T = np.array([[y, n - y] for y in range(n + 1)], dtype=np.int32)
        got, cnt, st = run(lofp, 2, [[(0, 1, th, ph)]], S, T)
        ref = np.array([oracle.bs_element(th, ph, x1, n - x1, y, n - y) for y in range(n + 1)])
        assert np.isfinite(got).all()
        ok, err = tol_ok(got, ref)
        assert ok, (n, err)
        assert (cnt == 1).all()
        assert abs(np.sum(np.abs(got) ** 2) - 1.0) < 1e-12


@pytest.mark.parametrize("D,k", [(3, k) for k in range(1, 11)] + [(4, 1), (4, 2), (4, 3)])
def test_density_workload(lofp, D, k):
    """10 modes, depth 3 and 4, S = T = (k,...,k), k = 1..10 (10..100 photons); the
    oracle path sum (pinned to Ryser at k <= 2) at every density it finishes in seconds."""
    M = 10
    layers = li.clements_mesh(M, D, seed=318 + D)
    S = np.full(M, k, dtype=np.int32)
    got, cnt, st = run(lofp, M, layers, S, S[None, :])
    ref, leaves = oracle.path_sum(M, layers, S, S[None, :], return_leaves=True)
    assert np.isfinite(got).all()
    ok, err = tol_ok(got, ref)
    assert ok, err
    assert np.array_equal(cnt, leaves)
    assert st["check_errors"] == 0


def test_density_workload_neighbours(lofp):
    """Density workload with outputs other than S (photons moved by one mode), depth 4."""
    M, D, k = 10, 4, 2
    layers = li.clements_mesh(M, D, seed=322)
    S = np.full(M, k, dtype=np.int32)
    rows = []
    for i in range(M - 1):
        t = S.copy()
        t[i] -= 1
        t[i + 1] += 1
        rows.append(t)
    T = np.array(rows, dtype=np.int32)
    got, cnt, _ = run(lofp, M, layers, S, T)
    ref, leaves = oracle.path_sum(M, layers, S, T, return_leaves=True)
    assert tol_ok(got, ref)[0]
    assert np.array_equal(cnt, leaves)


@pytest.mark.parametrize("seed", range(6))
def test_phase_gates(lofp, seed):
    """Linear and Kerr phase gates anywhere in random circuits against the oracle
    path sum with the same gates (pinned to a state-vector evolution)."""
    rng = np.random.default_rng(700 + seed)
    M = int(rng.integers(2, 8))
    D = int(rng.integers(1, 6))
    N = int(rng.integers(1, 6))
    layers = li.random_nn_circuit(M, D, rng, fill=0.9, reverse_prob=0.3)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    gates = [(int(rng.integers(0, M)), int(rng.integers(0, D + 1)), float(rng.uniform(-3, 3)),
              float(rng.uniform(-2, 2))) for _ in range(int(rng.integers(1, 8)))]
    T = li.all_outputs(M, N)
    if len(T) > 300:
        T = T[rng.choice(len(T), 300, replace=False)]
    got, cnt, _ = run(lofp, M, layers, S, T, gates)
    ref, leaves = oracle.path_sum(M, layers, S, T, return_leaves=True, gates=gates)
    ok, err = tol_ok(got, ref)
    assert ok, err
    assert np.array_equal(cnt, leaves)


def test_phase_gates_single_mode(lofp):
    """M = 1 has no cut to carry a gate: the gates multiply the single path."""
    gates = [(0, 0, 0.3, 0.1), (0, 2, -1.1, 0.05)]
    got, _, _ = run(lofp, 1, [[], []], [4], np.array([[4], [3]]), gates)
    want = np.exp(1j * (0.3 * 4 + 0.1 * 16)) * np.exp(1j * (-1.1 * 4 + 0.05 * 16))
    assert abs(got[0] - want) < 1e-15 and got[1] == 0


def test_gate_validation(lofp):
    with pytest.raises(lofp.LofpError) as e:
        lofp.Circuit(4, [[(0, 1, 0.1, 0.2)]], gates=[(4, 0, 0.1, 0.0)])
    assert e.value.status == 1
    with pytest.raises(lofp.LofpError) as e:
        lofp.Circuit(4, [[(0, 1, 0.1, 0.2)]], gates=[(0, 2, 0.1, 0.0)])
    assert e.value.status == 1


def _cfg4_slice(n=96):
    c = li.config(4)
    d = np.load(os.path.join(ROOT, "data", "cfg4.npz"))
    return c, d["T_cond"][:n].astype(np.int32), d["P_cond"][:n]


def test_bitwise_deterministic(lofp):
    """Fixed summation order (no floating-point atomics): two runs are bitwise equal."""
    c, T, P = _cfg4_slice()
    a1, _, _ = run(lofp, c.M, c.layers, c.S, T)
    a2, _, _ = run(lofp, c.M, c.layers, c.S, T)
    assert np.array_equal(a1.view(np.uint64), a2.view(np.uint64))


def test_cuda_graph_capture_and_replay(lofp):
    """lofp_amplitudes only enqueues work (no host sync, no device-to-host read), so it can
    be captured in a CUDA graph and replayed; replays give the same (bitwise) result."""
    c, T, P = _cfg4_slice(64)
    circ = lofp.Circuit(c.M, c.layers)
    Td = torch.from_numpy(T).cuda()
    out = torch.zeros((len(T), 2), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        circ.amplitudes(c.S, Td, out=out, stream=s)  # sizes the buffers, builds the tables
    torch.cuda.synchronize()
    first = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        circ.amplitudes(c.S, Td, out=out, stream=s)
    out.zero_()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, first)
    ref = oracle.amplitudes_permanent(c.M, c.layers, c.S, T[:4])
    assert tol_ok(torch.view_as_complex(out).cpu().numpy()[:4], ref)[0]


def test_stream_ordered_no_host_sync(lofp):
    """The call returns before its kernels finish: a long batch enqueued behind a long
    device sleep is still pending when the call returns, and the result is correct."""
    c, T, P = _cfg4_slice(256)
    circ = lofp.Circuit(c.M, c.layers)
    Td = torch.from_numpy(T).cuda()
    s = torch.cuda.Stream()
    circ.amplitudes(c.S, Td, stream=s)  # warm-up (buffers)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(2e8))  # ~0.1 s of device time before our kernels
        a = circ.amplitudes(c.S, Td, stream=s)
    assert not s.query()  # still running: the call did not wait for the stream
    s.synchronize()
    ref = oracle.amplitudes_permanent(c.M, c.layers, c.S, T[:4])
    assert tol_ok(a.cpu().numpy()[:4], ref)[0]
    # a bigger batch grows the buffers (stream-ordered: still no host synchronisation)
    c2, T2, P2 = _cfg4_slice(1024)
    Td2 = torch.from_numpy(T2).cuda()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(2e8))
        a2 = circ.amplitudes(c.S, Td2, stream=s)
    assert not s.query()
    s.synchronize()
    assert tol_ok(a2.cpu().numpy()[:256], a.cpu().numpy())[0]


def test_small_units(lofp, monkeypatch):
    """A small unit size splits every tree into many prefix units (the plan kernel's
    split, north_star 'splits the path tree ... into prefixes'); same paths, same values."""
    c, T, P = _cfg4_slice(48)
    base, _, _ = run(lofp, c.M, c.layers, c.S, T)
    monkeypatch.setenv("LOFP_UNIT_PATHS", "200000")
    got, cnt, st = run(lofp, c.M, c.layers, c.S, T)
    assert st["units"] > 10 * len(T)
    assert np.array_equal(cnt, P)
    assert tol_ok(got, base)[0]


def test_subsplits_when_lists_exceed_scratch(lofp, monkeypatch):
    """A 2 MiB scratch per block cannot hold the half-path lists of the larger configs[4]
    trees: units are split again inside the kernel (fixing one more column) and processed
    in turn; counts stay exact, values match the Ryser permanent."""
    c, T, P = _cfg4_slice(48)
    monkeypatch.setenv("LOFP_SLAB_MB", "2")
    monkeypatch.setenv("LOFP_UNIT_PATHS", str(1 << 40))
    got, cnt, st = run(lofp, c.M, c.layers, c.S, T)
    assert st["subsplits"] > 0
    assert np.array_equal(cnt, P)
    ref = oracle.amplitudes_permanent(c.M, c.layers, c.S, T[:6])
    assert tol_ok(got[:6], ref)[0]


def test_wrong_device_or_buffer_rejected(lofp):
    c, T, P = _cfg4_slice(4)
    circ = lofp.Circuit(c.M, c.layers)
    Td = torch.from_numpy(T).cuda()
    with pytest.raises(ValueError):
        circ.amplitudes(c.S, Td, out=torch.zeros((4, 2), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        circ.amplitudes(c.S, Td, out=torch.zeros((3, 2), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        circ.amplitudes(c.S, Td.cpu())


@pytest.mark.parametrize("idx,n,env", [(2, 256, {}), (3, 256, {}), (4, 256, {}),
                                       (3, 128, {"LOFP_UNIT_PATHS": "100000"}),
                                       (4, 96, {"LOFP_SLAB_MB": "2", "LOFP_UNIT_PATHS": str(1 << 40)})])
def test_debug_build_bounds_checks(lofp, idx, n, env):
    """compute-sanitizer is closed on this pool: the debug build (-DLOFP_DEBUG) checks every
    list, segment, context, schedule and unit-slot index on the device and traps with the
    failing site; conditioned slices, small units and forced sub-splits run clean."""
    import subprocess
    import sys
    from paper_2510_26408_b200 import _build
    assert os.path.exists(_build.DEBUG_LIB), "build() builds liblofp_debug.so"
    e = dict(os.environ, LOFP_LIB=_build.DEBUG_LIB, **env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "repro.py"), str(idx), str(n)], env=e,
                       capture_output=True, text=True, timeout=600)
    assert "LOFP_DEBUG" not in r.stdout + r.stderr, (r.stdout + r.stderr)[-2000:]
    assert r.returncode == 0, r.stderr[-2000:]
    ok = [l for l in r.stdout.splitlines() if l.startswith("ok")]
    assert ok and ok[0].endswith("True") and ok[0].split()[3] == "0"


def test_context_reuse_new_input_and_two_streams(lofp):
    """One context, calls with different inputs S (tables rebuilt per call) on two
    different streams back to back (the second waits for the first's buffers)."""
    rng = np.random.default_rng(11)
    M, D = 8, 5
    layers = li.clements_mesh(M, D, seed=12)
    circ = lofp.Circuit(M, layers)
    S1 = np.array([1, 0, 1, 0, 1, 0, 1, 0], dtype=np.int32)
    S2 = np.array([2, 0, 0, 1, 0, 0, 1, 1], dtype=np.int32)
    T1 = li.all_outputs(M, 4)
    T2 = li.all_outputs(M, 5)
    T1 = T1[rng.choice(len(T1), 200, replace=False)]
    T2 = T2[rng.choice(len(T2), 200, replace=False)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    Td1, Td2 = torch.from_numpy(T1).cuda(), torch.from_numpy(T2).cuda()
    torch.cuda.synchronize()  # (the copies ran on the default stream)
    a1 = circ.amplitudes(S1, Td1, stream=s1)
    a2 = circ.amplitudes(S2, Td2, stream=s2)
    a3 = circ.contract(S1, Td1, stream=s1)
    torch.cuda.synchronize()
    r1 = oracle.path_sum(M, layers, S1, T1)
    r2 = oracle.path_sum(M, layers, S2, T2)
    assert tol_ok(a1.cpu().numpy(), r1)[0]
    assert tol_ok(a2.cpu().numpy(), r2)[0]
    assert tol_ok(a3.cpu().numpy(), r1)[0]


def test_path_budget(lofp):
    """lofp_set_path_budget (SURVEY §5 failure guard): outputs above the budget are not
    enumerated (NaN, counted); the others are unchanged."""
    c, T, P = _cfg4_slice(96)
    circ = lofp.Circuit(c.M, c.layers)
    full, _, _ = run(lofp, c.M, c.layers, c.S, T)
    budget = int(np.median(P))
    circ.set_path_budget(budget)
    cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    a = circ.amplitudes(c.S, torch.from_numpy(T).cuda(), counts=cnt).cpu().numpy()
    st = circ.stats()
    over = P > budget
    assert st["over_budget"] == int(over.sum()) > 0
    assert np.isnan(a[over]).all()
    assert tol_ok(a[~over], full[~over])[0]  # (another batch total: other unit sizes, other rounding)
    assert np.array_equal(cnt.cpu().numpy()[~over].astype(np.uint64), P[~over])
    circ.set_path_budget(0)
    b = circ.amplitudes(c.S, torch.from_numpy(T).cuda()).cpu().numpy()
    assert np.array_equal(b, full)


def test_limits_modes_layers(lofp):
    """At the ABI limits: 128 modes (a 4-layer mesh, 10 photons) and 64 layers (a 4-mode
    circuit whose BS sit in every 8th layer), values against the oracle and Ryser."""
    rng = np.random.default_rng(128)
    M = 128
    layers = li.clements_mesh(M, 4, seed=128)
    S = np.zeros(M, dtype=np.int32)
    S[np.arange(0, 20, 2)] = 1
    T = li.displaced_patterns(M, [i for i in range(M) if S[i]], 3, 200, rng)[0]
    T = T[oracle.reachable(M, layers, S, T)][:40]
    assert len(T) >= 10
    got, cnt, st = run(lofp, M, layers, S, T)
    ref, leaves = oracle.path_sum(M, layers, S, T, return_leaves=True)
    assert tol_ok(got, ref)[0]
    assert np.array_equal(cnt, leaves)
    M, D = 4, 64  # 64 layers, every 8th carrying BS (a full 64-layer mesh has ~1e20 paths)
    full = li.clements_mesh(M, 8, seed=64)
    layers = [full[l // 8] if l % 8 == 0 else [] for l in range(D)]
    S = np.array([1, 1, 0, 1], dtype=np.int32)
    T = li.all_outputs(M, 3)
    got, cnt, st = run(lofp, M, layers, S, T)
    ref = oracle.amplitudes_permanent(M, layers, S, T)
    assert tol_ok(got, ref)[0]
    assert abs(np.sum(np.abs(got) ** 2) - 1) < 1e-12
