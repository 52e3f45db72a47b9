"""Per-output cost of the strip contraction (NEXT-1) on configs[3] as drawn: terms and
single-output kernel time of each output, against the batch call.  Diagnostic only."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit

c = li.config(3)
d = np.load(os.path.join(ROOT, "data", "cfg3.npz"))
T = d["T_literal"].astype(np.int32)
B = len(T)
circ = Circuit(c.M, c.layers)
dev = torch.device("cuda")
Td = torch.from_numpy(np.ascontiguousarray(T)).to(dev)
out = torch.empty((B, 2), dtype=torch.float64, device=dev)


def timed(Tx, o, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        circ.contract(c.S, Tx, out=o)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for _ in range(3):
    circ.contract(c.S, Td, out=out)
tb = timed(Td, out, 5)
st = circ.stats()
print(json.dumps({"batch_ms": tb, "terms": st["terms"], "states": st["max_states"]}))
terms = np.zeros(B)
ms = np.zeros(B)
o1 = torch.empty((1, 2), dtype=torch.float64, device=dev)
for b in range(B):
    Tb = Td[b:b + 1]
    ms[b] = timed(Tb, o1, 2)
    terms[b] = circ.stats()["terms"]
order = np.argsort(-terms)
print(json.dumps({"single_ms_max": ms.max(), "single_ms_median": float(np.median(ms)),
                  "terms_max": terms.max(), "terms_median": float(np.median(terms)), "terms_mean": terms.mean(),
                  "terms_sum": terms.sum(), "top10_terms": terms[order[:10]].tolist(),
                  "top10_ms": ms[order[:10]].tolist(),
                  "terms_quantiles": np.quantile(terms, [0.5, 0.9, 0.99, 0.999, 1]).tolist()}))
# batch without the 16 biggest outputs
keep = np.sort(order[16:])
Tk = Td[torch.from_numpy(keep).to(dev)].contiguous()
ok = torch.empty((len(keep), 2), dtype=torch.float64, device=dev)
print(json.dumps({"batch_minus_top16_ms": timed(Tk, ok, 5)}))
np.savez(os.path.join(ROOT, "gpurun_out", "contract_probe.npz"), terms=terms, ms=ms)
