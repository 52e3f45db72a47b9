"""Unit-kernel phase split (lofp_stats phase_cycles) on the conditioned batches."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit
NAMES = ["tail", "counts+split", "left lists", "right lists", "pairs+tables", "tiles", "tile wait", "fetch/setup/reduce"]
for idx in [int(x) for x in (sys.argv[1:] or ["4", "2", "3"])]:
    c = li.config(idx)
    d = np.load(os.path.join(ROOT, "data", f"cfg{idx}.npz"))
    T = torch.from_numpy(d["T_cond"].astype(np.int32)).cuda()
    circ = Circuit(c.M, c.layers)
    for _ in range(2):
        circ.amplitudes(c.S, T)
    torch.cuda.synchronize()
    st = circ.stats()
    ph = np.array(st["phase_cycles"], dtype=np.float64)
    tot = ph.sum()
    print(f"cfg{idx}: units_ms {st['units_ms']:.1f} paths/s {st['paths'] / st['units_ms'] * 1e3:.3e} units {st['units']} "
          f"pairs {st['pairs']} elements {st['elements']}")
    print("   " + "  ".join(f"{n} {100 * v / tot:.1f}%" for n, v in zip(NAMES, ph)))
    # block time accounted by the phases over grid x kernel time (the rest: blocks that ran out of units)
    print(f"   blocks busy {tot / (st['grid_blocks'] * st['units_ms'] * 1e-3 * 1.965e9):.3f} of grid x kernel time")
    tc = st["tile_cycles"]
    print(f"   tiles: staging {100 * tc[0] / max(1, tc[0] + tc[1]):.1f}% of warp tile time")
if os.environ.get("HERO"):
    c = li.config(4)
    d = np.load(os.path.join(ROOT, "data", "cfg4.npz"))
    T = torch.from_numpy(d["T_hero"].astype(np.int32)).cuda()
    circ = Circuit(c.M, c.layers)
    for _ in range(2):
        circ.amplitudes(c.S, T)
    torch.cuda.synchronize()
    st = circ.stats()
    print(f"hero: units_ms {st['units_ms']:.1f} paths/s {st['paths'] / st['units_ms'] * 1e3:.3e} units {st['units']}")
