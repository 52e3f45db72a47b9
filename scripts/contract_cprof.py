"""Phase clocks and level statistics of the contraction warp kernel (liblofp_cprof.so, built with
-DLOFP_CPROF) on configs[3] as drawn.  Diagnostic only."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit

c = li.config(3)
T = np.load(os.path.join(ROOT, "data", "cfg3.npz"))["T_literal"].astype(np.int32)
circ = Circuit(c.M, c.layers)
Td = torch.from_numpy(np.ascontiguousarray(T)).cuda()
out = torch.empty((len(T), 2), dtype=torch.float64, device="cuda")
circ.contract(c.S, Td, out=out)
torch.cuda.synchronize()
st = circ.stats()
ph = list(st["phase_cycles"])
names = ["setup_clk", "levelrows_clk", "entries_clk", "-", "entries", "sum_batch_max_row", "sum_rows", "cuts"]
d = dict(zip(names, ph))
d["terms"] = st["terms"]
d["avg_row"] = ph[6] / max(ph[4], 1)
d["lane_util_rows"] = ph[6] / max(32 * ph[5], 1)
d["entries_per_cut"] = ph[4] / max(ph[7], 1)
d["clk_per_cut_entries"] = ph[2] / max(ph[7], 1)
d["clk_per_cut_levelrows"] = ph[1] / max(ph[7], 1)
d["setup_clk_per_output"] = ph[0] / len(T)
print(json.dumps(d))
