import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lofp_inputs as li, oracle
from paper_2510_26408_b200 import Circuit
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rng = np.random.default_rng(4200 + seed)
M = int(rng.integers(18, 23)); D = int(rng.integers(3, 5))
layers = li.clements_mesh(M, D, seed=100 + seed)
N = int(rng.integers(M // 2 + 2, M - 3))
S = np.zeros(M, dtype=np.int32); S[np.sort(rng.choice(M, N, replace=False))] = 1
T = li.uniform_subsets(M, N, 4000, rng)
T = T[oracle.reachable(M, layers, S, T)]
P = np.array(oracle.count_paths(M, layers, S, T), dtype=object)
T = T[(P > 0) & (P <= 3 * 10 ** 5)][:150]
print("M D N B", M, D, N, len(T), flush=True)
for n in (1, 2, 8, len(T)):
    c = Circuit(M, layers)
    cnt = torch.zeros(n, dtype=torch.int64, device="cuda")
    a = c.amplitudes(S, torch.from_numpy(np.ascontiguousarray(T[:n])).cuda(), counts=cnt)
    torch.cuda.synchronize()
    st = c.stats()
    ref, leaves = oracle.path_sum(M, layers, S, T[:n], return_leaves=True)
    print(n, "maxerr", float(np.abs(a.cpu().numpy() - ref).max()), "counts ok", np.array_equal(cnt.cpu().numpy().astype(np.uint64), leaves),
          {k: st[k] for k in ("chains", "chain_fallbacks", "levels", "max_factors")}, flush=True)
