"""Per source line of one ncu --set full capture: share of warp instructions and active lanes
(Thread Instructions Executed / Instructions Executed).

usage: python scripts/ncu_lanes.py <report.ncu-rep> <liblofp.so> <kernel (mangled substring)> <source file in csrc/>
"""
import csv, subprocess, sys, re, collections, os, tempfile
rep, so, kern, src = sys.argv[1:5]
so = os.path.abspath(so)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cub = sorted(f for f in os.listdir(tmp) if f.endswith(".cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
st = next(i for i, l in enumerate(dis) if ".text." in l and kern in l and l.lstrip().startswith(".section"))
seq = []; cur = 0
for l in dis[st + 1:]:
    if l.lstrip().startswith(".section"): break
    m = re.search(r'## File ".*/(\w+\.\w+)", line (\d+)', l)
    if m:
        cur = int(m.group(2)) if m.group(1) == src else cur; continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[A-Z@{]", l): seq.append(cur)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(out)); hdr = r[1]; rows = r[2:]
iE = hdr.index("Instructions Executed"); iT = hdr.index("Thread Instructions Executed")
ex = collections.Counter(); th = collections.Counter()
for ln, x in zip(seq, rows):
    ex[ln] += int(x[iE] or 0); th[ln] += int(x[iT] or 0)
lines = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2510_26408_b200", "csrc", src)).read().split("\n")
tot = sum(ex.values())
for ln, v in ex.most_common(25):
    print(f"{100*v/tot:5.1f}%  lanes {th[ln]/max(v,1):5.1f}  line {ln:4d} {lines[ln-1].strip()[:80] if ln else ''}")
