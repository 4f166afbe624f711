"""Per-source-line executed instructions (and their top opcodes) of an ncu
`--set full --import-source on` capture; the kernels are built with -lineinfo.

python tools/src_hotspots.py REP [N]
"""
import csv, sys, subprocess
from collections import defaultdict
raw = subprocess.run(["ncu","-i",sys.argv[1],"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
import io
rows=list(csv.reader(io.StringIO(raw)))
cur=None; data=[]; ops=defaultdict(lambda: defaultdict(float)); line=None
for r in rows:
    if not r: continue
    if r[0]=='File Path': cur=r[1].split('/')[-1]; continue
    if r[0] in ('Function Name','Line No'): continue
    if r[0]!='':
        line=(cur,r[0],r[1][:90])
        try: n=float(r[7].replace(',','') or 0)
        except: n=0
        data.append((n,line))
    else:
        op=r[3].split()
        if not op: continue
        o=op[1] if op[0].startswith('@') else op[0]
        try: n=float(r[7].replace(',','') or 0)
        except: n=0
        ops[line][o.split('.')[0]]+=n
tot=sum(d[0] for d in data)
print("total", tot)
for n,l in sorted(data,reverse=True)[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    top=sorted(ops[l].items(),key=lambda x:-x[1])[:4]
    print(f"{100*n/tot:5.1f}% {l[0]}:{l[1]} {l[2][:60]:60s} "+" ".join(f"{k}:{100*v/n:.0f}" for k,v in top))
