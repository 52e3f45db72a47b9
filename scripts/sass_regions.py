"""Map the per-instruction counts of an ncu source-page dump (scripts/summarize_ncu.py's
hot list) onto source regions of the chain-mode enumeration kernel (line ranges of
lofp_kernels.cu; needs nvdisasm -g output of the same build in /tmp/all2.txt)."""
import re,collections
Ls=open('/tmp/all2.txt').read().split('\n')
tag='ILb0ELb1ELb0E'
st=[i for i,l in enumerate(Ls) if l.startswith('//---') and tag in l and '.text' in l][0]
en=next(i for i in range(st+1,len(Ls)) if Ls[i].startswith('//---------------------'))
last=None; seq=[]
for l in Ls[st:en]:
    m=re.search(r'## File ".*/(\w+\.\w+)", line (\d+)',l)
    if m:
        if m.group(1)=='lofp_kernels.cu' and int(m.group(2))>430: last=int(m.group(2))
        continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+[A-Z@{]',l): seq.append(last or 0)
rows=[l for l in open('/tmp/hot_r1g.txt')]
assert len(seq)==len(rows), (len(seq), len(rows))
def phase(n):
    if n < 523: return 'prologue/helpers'
    if n < 583: return 'acquire + plan staging'
    if n < 672: return 'item start'
    if n < 741: return 'hand-over'
    if n < 832: return 'walk step'
    if n < 1022: return 'chain ranges (+ short-chain batch)'
    if n < 1065: return 'pair table W'
    if n < 1099: return 'split + prefix digits'
    if n < 1129: return 'suffix table'
    if n < 1194: return 'prefix products + paths'
    if n < 1204: return 'resume walk'
    if n < 1241: return 'queue feeding'
    return 'item end'
ex=collections.Counter(); stl=collections.Counter(); nin=collections.Counter()
for a,l in zip(seq,rows):
    p=phase(a); v=float(l.split()[1]); ex[p]+=v; stl[p]+=float(re.search(r"st\s*([0-9.]+)",l).group(1)); nin[p]+=1
print(f"{'region':38s} {'instr %':>8s} {'stall %':>8s} {'SASS':>6s}")
for p in sorted(ex, key=lambda k:-ex[k]):
    print(f"{p:38s} {ex[p]/10:8.1f} {stl[p]/10:8.1f} {nin[p]:6d}")
