"""Small reproducer: a slice of a conditioned batch through the path-sum call (debug aid)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
c = li.config(idx)
d = np.load(os.path.join(ROOT, "data", f"cfg{idx}.npz"))
T = torch.from_numpy(d["T_cond"][:n].astype(np.int32)).cuda()
cnt = torch.zeros(n, dtype=torch.int64, device="cuda")
circ = Circuit(c.M, c.layers)
a = circ.amplitudes(c.S, T, counts=cnt)
torch.cuda.synchronize()
st = circ.stats()
print("ok", st["units"], st["subsplits"], st["check_errors"], bool((cnt.cpu().numpy().astype(np.uint64) == d["P_cond"][:n]).all()))
