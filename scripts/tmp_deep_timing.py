import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit
M, D = 6, 16
layers = li.clements_mesh(M, D, seed=1616)
S = np.array([1, 1, 1, 0, 0, 0], dtype=np.int32)
T = torch.from_numpy(li.all_outputs(M, 3)[:int(sys.argv[1])]).cuda()
c = Circuit(M, layers)
t0 = time.time()
a = c.amplitudes(S, T); torch.cuda.synchronize()
st = c.stats()
print(f"B={len(T)} {time.time()-t0:.1f} s", {k: st[k] for k in ("unsupported", "generic", "total_ms", "cmuls", "paths")}, flush=True)
