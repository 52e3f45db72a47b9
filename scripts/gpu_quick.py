"""Quick GPU smoke/debug: configs[0..1] and random circuits against the oracle."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import lofp_inputs as li
import oracle
from paper_2510_26408_b200 import Circuit


def run(M, layers, S, T, gates=()):
    c = Circuit(M, layers, gates)
    Td = torch.from_numpy(np.ascontiguousarray(T, dtype=np.int32)).cuda()
    cnt = torch.zeros(len(T), dtype=torch.int64, device="cuda")
    a = c.amplitudes(S, Td, counts=cnt)
    torch.cuda.synchronize()
    return a.cpu().numpy(), cnt.cpu().numpy(), c.stats()


def check(name, got, ref, cnt=None, leaves=None, st=None):
    err = np.abs(got - ref)
    ok = (err <= 1e-12 + 1e-9 * np.abs(ref)).all()
    cok = True if cnt is None else np.array_equal(cnt.astype(np.uint64), leaves.astype(np.uint64))
    print(f"{name}: ok={ok} maxerr={err.max() if err.size else 0:.2e} counts_ok={cok} "
          f"stats={ {k: st[k] for k in ('paths','units','pairs','elements','check_errors','unsupported','max_list','units_ms')} if st else ''}",
          flush=True)
    return ok and cok


allok = True
c = li.config(0)
T = c.draw_outputs()
got, cnt, st = run(c.M, c.layers, c.S, T)
ref, leaves = oracle.path_sum(c.M, c.layers, c.S, T, return_leaves=True)
allok &= check("cfg0", got, ref, cnt, leaves, st)
for seed in range(int(os.environ.get("NRAND", "30"))):
    rng = np.random.default_rng(9000 + seed)
    M = int(rng.integers(1, 10)); D = int(rng.integers(0, 8)); N = int(rng.integers(0, 6))
    layers = li.random_nn_circuit(M, D, rng, fill=float(rng.uniform(0.4, 1.0)), reverse_prob=0.4)
    S = np.zeros(M, dtype=np.int32)
    for m in rng.integers(0, M, size=N):
        S[m] += 1
    T = li.all_outputs(M, N)
    if len(T) > 300:
        T = T[rng.choice(len(T), 300, replace=False)]
    T = np.concatenate([T, np.clip(T[:3] + 1, 0, None)])
    got, cnt, st = run(M, layers, S, T)
    ref, leaves = oracle.path_sum(M, layers, S, T, return_leaves=True)
    r = check(f"rand{seed} M={M} D={D} N={N}", got, ref, cnt, leaves, st)
    allok &= r
c = li.config(1)
d = np.load(os.path.join(ROOT, "data", "cfg1.npz"))
T = d["T_literal"].astype(np.int32)
got, cnt, st = run(c.M, c.layers, c.S, T)
ref = oracle.path_sum(c.M, c.layers, c.S, T)
allok &= check("cfg1", got, ref, cnt, d["P_literal"], st)
for idx in (2, 3, 4):
    c = li.config(idx)
    d = np.load(os.path.join(ROOT, "data", f"cfg{idx}.npz"))
    T = d["T_cond"].astype(np.int32)
    n = int(os.environ.get("NCOND", "256"))
    t0 = time.time()
    got, cnt, st = run(c.M, c.layers, c.S, T[:n])
    print(f"cfg{idx} cond[:{n}] wall {time.time()-t0:.2f}s paths/s(units) {st['paths']/max(st['units_ms'],1e-9)*1e3:.3e}", flush=True)
    small = np.argsort(d["P_cond"][:n])[:6]
    ref = oracle.path_sum(c.M, c.layers, c.S, T[:n][small])
    allok &= check(f"cfg{idx} small", got[small], ref, cnt, d["P_cond"][:n], st)
print("ALL OK" if allok else "FAILURES")
