"""Quick GPU throughput probe (development aid, not the bench): times lofp_amplitudes on a
prefix of each config's batch sized to a path budget."""
import os, sys, time, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 2e10
cfgs = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [1, 2, 3, 4]
for idx in cfgs:
    c = li.config(idx)
    d = np.load(os.path.join(ROOT, "data", f"cfg{idx}.npz"))
    T = (d["T_cond"] if "T_cond" in d.files else d["T_literal"]).astype(np.int32)
    P = (d["P_cond"] if "P_cond" in d.files else d["P_literal"]).astype(np.float64)
    if os.environ.get("PROBE_SMALLEST"):  # the smallest trees first: many outputs, short run
        o = np.argsort(P, kind="stable")
        T, P = T[o], P[o]
    n = int(np.searchsorted(np.cumsum(P), budget)) if P.sum() > budget else len(P)
    n = max(n, 1)
    T, P = T[:n], P[:n]
    circ = Circuit(c.M, c.layers)
    Td = torch.from_numpy(T).cuda()
    circ.amplitudes(c.S, Td[: min(n, 64)]); torch.cuda.synchronize()
    res = []
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); a = circ.amplitudes(c.S, Td); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1); st = circ.stats()
        res.append(ms)
    if os.environ.get("PROBE_HIST"):
        cnt = torch.zeros(n, dtype=torch.int64, device="cuda")
        circ.amplitudes(c.S, Td, counts=cnt); torch.cuda.synchronize()
        h, sp = circ.work_histograms()
        pc = circ.phase_cycles().astype(float)
        names = ["dfs", "ranges", "Wbuild", "split+digits", "paths", "return+feed", "acquire", "suffix"]
        print("phase cycles %:", {n: round(100 * x / pc.sum(), 1) for n, x in zip(names, pc)})
        print("handover by leaf-distance:", h[:40].tolist())
        print("spill by leaf-distance:", sp[:40].tolist())
    print(json.dumps(dict(cfg=idx, outputs=n, paths=P.sum(), ms=min(res), paths_per_s=P.sum() / (min(res) * 1e-3),
                          enum_ms=st["enum_ms"], total_ms=st["total_ms"], items=st["items"], spills=st["spills"], donations=st["donations"], ovf=st["overflows"], block=st["block_threads"], maxF=st["max_factors"], maxS=st["max_scatter"], chains=st["chains"], chain_fb=st["chain_fallbacks"],
                          levels=st["levels"], entries=st["table_entries"], smem=st["smem_bytes"], grid=st["grid_blocks"])), flush=True)
