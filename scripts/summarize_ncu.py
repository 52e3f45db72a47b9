"""Summarise one ncu --set full capture (.ncu-rep): headline metrics, warp-stall split,
SASS opcode mix and (for lofp_units_kernel / lofp_contract_kernel) the per-function split.

usage: python scripts/summarize_ncu.py <report.ncu-rep> [kernel-name]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kernel = sys.argv[2] if len(sys.argv) > 2 else "lofp_units_kernel"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(raw))
d = dict(zip(r[0], r[2]))
units = dict(zip(r[0], r[1]))
print(f"report: {rep}")
print(f"kernel: {d.get('Kernel Name')}  grid {d.get('launch__grid_size')} x block {d.get('launch__block_size')}")
for k in ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "launch__occupancy_limit_registers",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__t_sector_hit_rate.pct",
          "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]:
    if k in d:
        print(f"  {k:78s} {d[k]} {units.get(k, '')}")
import re
for k in sorted(d):  # the memory pipes: which unit is closest to its peak
    if re.match(r"((l1tex__throughput|lts__throughput|sm__throughput|l1tex__lsu_writeback_active|"
                r"sm__memory_throughput)\.avg\.pct_of_peak_sustained_elapsed$|"
                r"l1tex__data_pipe_lsu_wavefronts\.sum\.pct_of_peak_sustained_elapsed$|"
                r"l1tex__t_(requests|sectors)_pipe_lsu_mem_global_op_ld\.sum$)", k):
        print(f"  {k:78s} {d[k]} {units.get(k, '')}")
dfma = d.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")
cyc = d.get("sm__cycles_elapsed.avg")
if dfma and cyc:
    print(f"  DFMA lane-ops per launch (derived)                                             "
          f"{float(dfma) * float(cyc):.4e}")
st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and
      not k.endswith("not_issued") and v]
tot = sum(v for _, v in st) or 1
print("  stalls: " + ", ".join(f"{k[33:]} {100 * v / tot:.1f}%" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rr = list(csv.reader(src))
hdr, rows = rr[1], rr[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
c = collections.Counter()
te = 0
for x in rows:
    e = int(x[iE] or 0)
    op = x[iS].strip().split()
    if not op:
        continue
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    c[o] += e
    te += e
print("  opcode mix: " + ", ".join(f"{k} {100 * v / te:.1f}%" for k, v in c.most_common(14)))
