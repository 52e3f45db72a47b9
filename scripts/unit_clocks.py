"""Experiment (liblofp_uclk.so, -DLOFP_UNIT_CLOCKS): per-unit duration and end time of the
unit kernel on a conditioned batch whose outputs are one unit each."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import lofp_inputs as li
from paper_2510_26408_b200 import Circuit
idx = int(sys.argv[1])
c = li.config(idx)
d = np.load(os.path.join(ROOT, "data", f"cfg{idx}.npz"))
P = d["P_cond"].astype(np.float64)
T = torch.from_numpy(d["T_cond"].astype(np.int32)).cuda()
circ = Circuit(c.M, c.layers)
for _ in range(2):
    a = circ.amplitudes(c.S, T)
torch.cuda.synchronize()
a = a.cpu().numpy(); a = np.stack([a.real, a.imag], axis=1) if np.iscomplexobj(a) else a
cyc = np.floor(a[:, 0]); blk = np.round((a[:, 0] - cyc) * 1024).astype(int); end = a[:, 1]
t0 = (end - cyc / 1.965).min(); end = (end - t0) * 1e-6  # ms
dur = cyc / 1.965e6  # ms
print(f"cfg{idx}: kernel end {end.max():.1f} ms; units {len(P)}")
rate = P / dur / 1e6  # paths per ns... (1e9 paths/s)
big = P > 2 ** 27
print("  rate of units > 2^27 paths (1e9 paths/s per block): quantiles", np.round(np.quantile(rate[big] / 1e3, [0, .1, .5, .9, 1]), 2))
last = np.zeros(blk.max() + 1); nlast = np.zeros(blk.max() + 1)
for b in range(blk.max() + 1):
    m = blk == b
    if m.any():
        i = np.argmax(np.where(m, end, -1)); last[b] = end[i]; nlast[b] = P[i]
print("  block finish times (ms): quantiles", np.round(np.quantile(last, [0, .1, .5, .9, 1]), 1))
o = np.argsort(-last)[:10]
print("  last blocks: finish, last unit's paths, its duration, start of that unit")
for b in o:
    m = blk == b; i = np.argmax(np.where(m, end, -1))
    print(f"    block {b}: {last[b]:.1f} ms, P {P[i]:.2e}, {dur[i]:.1f} ms, started {end[i] - dur[i]:.1f} ms; units of the block {m.sum()}, paths {P[m].sum():.3e}")
print("  paths per block: quantiles", np.quantile([P[blk == b].sum() for b in range(blk.max() + 1)], [0, .1, .5, .9, 1]))
np.savez(os.path.join(ROOT, "gpurun_out", f"unit_clocks_cfg{idx}.npz"), P=P, dur=dur, end=end, blk=blk)
