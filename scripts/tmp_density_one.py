import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit
M, D, k = 10, 4, 10
layers = li.clements_mesh(M, D, seed=318 + D)
S = np.full(M, k, dtype=np.int32)
T = torch.from_numpy(S[None, :].copy()).cuda()
c = Circuit(M, layers)
for _ in range(2):
    c.amplitudes(S, T)
torch.cuda.synchronize()
print(c.stats()["total_ms"])
