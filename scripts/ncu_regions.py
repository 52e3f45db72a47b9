"""Attribute an ncu --set full capture of lofp_units_kernel to source functions.

usage: python scripts/ncu_regions.py <report.ncu-rep> [liblofp.so] [kernel] [source file in csrc/]
Pairs the report's per-SASS-instruction counters (program order) with the
nvdisasm -g line info of the same build, then sums executed instructions, FP64
instructions and warp-stall samples per device function of lofp_kernels.cu.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep = sys.argv[1]
so = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(__file__), "..", "paper_2510_26408_b200",
                                                         "liblofp.so")
src_path = os.path.join(os.path.dirname(__file__), "..", "paper_2510_26408_b200", "csrc",
                        sys.argv[4] if len(sys.argv) > 4 else "lofp_kernels.cu")
SRC = os.path.basename(src_path)
KERNEL = sys.argv[3] if len(sys.argv) > 3 else "lofp_units_kernel"

# function line ranges of lofp_kernels.cu
lines = open(src_path).read().split("\n")
starts = []
for i, l in enumerate(lines, start=1):
    m = re.match(r"^(?:__device__|__global__|static __device__)[^(]*?\b(\w+)\s*\(", l)
    if m:
        starts.append((i, m.group(1)))
starts.sort()


def func_of(line):
    name = "?"
    for s, n in starts:
        if s <= line:
            name = n
        else:
            break
    return name


tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cubins = sorted(f for f in os.listdir(tmp) if f.endswith(".cubin") and "host" not in f)
# the library holds one cubin per .cu file: take the one with the kernel's .text section
for cb in cubins:
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cb)], capture_output=True, text=True).stdout
    L = dis.split("\n")
    st = next((i for i, l in enumerate(L) if ".text." in l and KERNEL in l and l.lstrip().startswith(".section")), None)
    if st is not None:
        break
else:
    sys.exit(f"no .text section of {KERNEL} in {so}")
seq = []
cur = 0
for l in L[st + 1:]:
    if l.lstrip().startswith(".section"):
        break
    m = re.search(r'## File ".*/(\w+\.\w+)", line (\d+)', l)
    if m:
        cur = int(m.group(2)) if m.group(1) == SRC else cur
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[A-Z@{]", l):
        seq.append(cur)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
r = list(csv.reader(out))
hdr = r[1]
rows = r[2:]
iS, iE, iSt = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(os.environ.get("STALL_COL", "Warp Stall Sampling (All Samples)"))
if len(seq) != len(rows):
    print(f"warning: {len(seq)} SASS lines in the build vs {len(rows)} in the report", file=sys.stderr)
ex = collections.Counter()
fp = collections.Counter()
stl = collections.Counter()
byline = collections.Counter()
for ln, x in zip(seq, rows):
    f = func_of(ln)
    e = int(x[iE] or 0)
    ex[f] += e
    stl[f] += int(x[iSt] or 0)
    byline[(f, ln)] += int(x[iSt] or 0)
    op = x[iS].strip().split()
    o = (op[1] if op and op[0].startswith("@") else (op[0] if op else "")).split(".")[0]
    if o in ("DFMA", "DMUL", "DADD"):
        fp[f] += e
te, ts = sum(ex.values()), sum(stl.values())
print(f"{'function':22s} {'instr%':>7s} {'fp64%':>7s} {'stall%':>7s}")
for f in sorted(ex, key=lambda k: -stl[k]):
    print(f"{f:22s} {100 * ex[f] / te:7.1f} {100 * fp[f] / max(1, sum(fp.values())):7.1f} {100 * stl[f] / ts:7.1f}")
print("hottest lines (stall samples):")
for (f, ln), v in byline.most_common(12):
    print(f"  {100 * v / ts:5.1f}%  line {ln:5d} {f:18s} {lines[ln - 1].strip()[:80] if ln else ''}")
print("hottest lines (instructions executed):")
exl = collections.Counter()
for ln, x in zip(seq, rows):
    exl[ln] += int(x[iE] or 0)
for ln, v in exl.most_common(16):
    print(f"  {100 * v / te:5.1f}%  line {ln:5d} {lines[ln - 1].strip()[:90] if ln else ''}")
