"""Randomised cross-check of every GPU method against the oracle: 100 random circuits (local
and non-local pairs, partial layers, reversed pairs, phase gates, bunched inputs), every
output pattern (or a sample); the path sum (with exact path-product counts), the strip
contraction and the distribution call must all agree with the oracle path sum.
Tolerance (BASELINE.json north_star): |a - a_ref| <= 1e-12 + 1e-9 |a_ref|."""
import numpy as np
import pytest

import lofp_inputs as li
import oracle

pytestmark = pytest.mark.gpu
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


@pytest.mark.parametrize("block", range(4))
def test_fuzz(lofp, block):
    failures = []
    for seed in range(25 * block, 25 * block + 25):
        rng = np.random.default_rng(77000 + seed)
        M = int(rng.integers(1, 9))
        D = int(rng.integers(0, 6))
        N = int(rng.integers(0, 6))
        nonlocal_ = bool(rng.random() < 0.4) and M >= 3
        if nonlocal_:
            layers = li.random_nonlocal_circuit(M, D, rng, fill=float(rng.uniform(0.3, 1.0)))
        else:
            layers = li.random_nn_circuit(M, D, rng, fill=float(rng.uniform(0.3, 1.0)), reverse_prob=0.4)
        S = np.zeros(M, dtype=np.int32)
        for m in rng.integers(0, M, size=N):
            S[m] += 1
        gates = [(int(rng.integers(0, M)), int(rng.integers(0, D + 1)), float(rng.uniform(-3, 3)),
                  float(rng.uniform(-1, 1))) for _ in range(int(rng.integers(0, 3)))]
        T = li.all_outputs(M, N)
        if len(T) > 120:
            T = T[rng.choice(len(T), 120, replace=False)]
        prune = oracle.PRUNE_CONE if nonlocal_ else oracle.PRUNE_BOX
        ref, leaves = oracle.path_sum(M, layers, S, T, prune=prune, return_leaves=True, gates=gates)
        circ = lofp.Circuit(M, layers, gates)
        Td = torch.from_numpy(np.ascontiguousarray(T, dtype=np.int32)).cuda()
        cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda")
        a = circ.amplitudes(S, Td, counts=cnt).cpu().numpy()
        b = circ.contract(S, Td).cpu().numpy()
        st = circ.stats()
        Tall, d = circ.distribution(S)
        d = d.cpu().numpy()
        ok_a = tol_ok(a, ref)[0] and np.array_equal(cnt.cpu().numpy().astype(np.uint64), leaves)
        ok_b = tol_ok(b, ref)[0]
        ok_d = abs(np.sum(np.abs(d) ** 2) - 1.0) < 1e-12 if N <= 5 else True
        if not (ok_a and ok_b and ok_d and st["check_errors"] == 0):
            failures.append((seed, M, D, N, nonlocal_, ok_a, ok_b, ok_d))
    assert not failures, failures
