"""Summarise one ncu --set full capture (.ncu-rep) of the enumeration kernel: headline
metrics, warp-stall split, SASS opcode mix; optional per-instruction hot list (argv[2])."""
import csv, sys, subprocess
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout.splitlines()
r=list(csv.reader(raw)); hdr=r[0]; vals=r[2]; d=dict(zip(hdr,vals))
for k in ['gpu__time_duration.sum','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','smsp__thread_inst_executed_per_inst_executed.ratio','smsp__inst_executed.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','launch__registers_per_thread']:
    print(f"{k:75s} {d.get(k)}")
stalls=[(h,v) for h,v in d.items() if 'smsp__pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued')]
tot=sum(float(v) for h,v in stalls if v)
print(' '.join(f"{h[33:]}={float(v)/tot*100:.1f}%" for h,v in sorted(stalls,key=lambda x:-float(x[1] or 0))[:8]))
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout.splitlines()
r=list(csv.reader(src)); hdr=r[1]; rows=r[2:]
iS=hdr.index("Source"); iE=hdr.index("Instructions Executed"); iA=hdr.index("Address"); iT=hdr.index("Avg. Threads Executed"); iSt=hdr.index("Warp Stall Sampling (All Samples)")
from collections import Counter
c=Counter(); tot=0
for x in rows:
    e=int(x[iE]); op=x[iS].strip().split()
    if not op: continue
    o=op[1] if op[0].startswith('@') else op[0]
    c[o.split('.')[0]]+=e; tot+=e
print([(k,round(v/tot*100,1)) for k,v in c.most_common(24)])
if len(sys.argv)>2:
    stot=sum(int(x[iSt]) for x in rows)
    with open(sys.argv[2],'w') as f:
        for x in rows:
            f.write(f"{x[iA][-5:]} {int(x[iE])/tot*1000:7.3f} st{int(x[iSt])/stot*1000:6.2f} thr{float(x[iT]):5.1f}  {x[iS].strip()[:100]}\n")
