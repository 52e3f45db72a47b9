"""The paper's scaling experiments re-run on one B200 with our own seeded meshes (the paper's
circuit parameters are unpublished; its figures are not in the text):
  * P:315-328 (fig. Higher_photons): 10 modes, depth 3 and 4, S = T = (k,...,k), k = 1..10 --
    the exact path count, the path-sum time and the contraction time per amplitude;
  * P:237-252 (fig. linear_time): 1 photon per mode, depth 3..5, M = 20..120 -- contraction
    time per amplitude against M (the paper: linear in M).
Prints one JSON object (also written to the path given as argv[1])."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lofp_inputs as li  # noqa: E402
from paper_2510_26408_b200 import Circuit  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"density": [], "linear_in_M": []}
for D in (3, 4):
    M = 10
    layers = li.clements_mesh(M, D, seed=318 + D)
    circ = Circuit(M, layers)
    for k in range(1, 11):
        S = np.full(M, k, dtype=np.int32)
        T = torch.from_numpy(S[None, :].copy()).cuda()
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        a = circ.amplitudes(S, T, counts=cnt)
        torch.cuda.synchronize()
        P = int(cnt.item()) & 0xFFFFFFFFFFFFFFFF
        t_path = timed(lambda: circ.amplitudes(S, T), reps=3 if P > 1e10 else 5)
        t_con = timed(lambda: circ.contract(S, T))
        out["density"].append({"D": D, "k": k, "photons": 10 * k, "paths": P, "path_sum_ms": t_path,
                               "paths_per_s": P / (t_path * 1e-3), "contraction_ms": t_con,
                               "amplitude": [float(a[0].real), float(a[0].imag)]})
for D in (3, 4, 5):
    for M in (20, 40, 60, 80, 100, 120):
        layers = li.clements_mesh(M, D, seed=247 + D)
        S = np.ones(M, dtype=np.int32)
        T = torch.from_numpy(S[None, :].copy()).cuda()
        circ = Circuit(M, layers)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        circ.contract(S, T, counts=cnt)
        torch.cuda.synchronize()
        P = int(cnt.item()) & 0xFFFFFFFFFFFFFFFF  # (uint64; 2^64 - 1 = saturated)
        out["linear_in_M"].append({"D": D, "M": M, "paths": P if P < 2 ** 64 - 1 else ">= 1.8e19",
                                   "contraction_ms": timed(lambda: circ.contract(S, T))})
s = json.dumps(out)
print(s)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(s + "\n")
