"""P:318 density workload (10 modes, depth 4, S = T = (k,...,k)) single outputs: path-sum
statistics per unit-size setting (units, pairs, list elements, phase split, tile staging share)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit
M, D = 10, 4
layers = li.clements_mesh(M, D, seed=318 + D)
for k in (8, 10):
    S = np.full(M, k, dtype=np.int32)
    T = torch.from_numpy(S[None, :].copy()).cuda()
    c = Circuit(M, layers)
    for upb in ("2", "8", "32"):
        os.environ["LOFP_UNITS_PER_BLOCK"] = upb
        c.amplitudes(S, T); torch.cuda.synchronize()
        for _ in range(2): c.amplitudes(S, T)
        torch.cuda.synchronize()
        st = c.stats()
        ph = np.array(st["phase_cycles"], float); tc = np.array(st["tile_cycles"], float)
        print(f"k={k} upb={upb} units_ms={st['units_ms']:.2f} total_ms={st['total_ms']:.2f} paths={st['paths']:.3e} "
              f"rate={st['paths']/st['units_ms']/1e9:.3e} units={st['units']} pairs={st['pairs']} elems={st['elements']} "
              f"maxlist={st['max_list']} states={st['max_states']} phases%={np.round(100*ph/ph.sum(),1).tolist()} "
              f"tile stage/fma={tc[0]/max(tc.sum(),1):.3f}", flush=True)
