"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump by source line."""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[2]; data=rows[3:]
idx=hdr.index('Warp Stall Sampling (All Samples)')
ex=hdr.index('Instructions Executed')
agg=collections.defaultdict(float); src={}; inst=collections.defaultdict(float)
cur=None
for r in data:
    if len(r)<len(hdr): continue
    if r[0]: cur=r[0]; src[cur]=r[1]
    try: agg[cur]+=float(r[idx] or 0); inst[cur]+=float(r[ex] or 0)
    except: pass
tot=sum(agg.values())
for ln,v in sorted(agg.items(), key=lambda x:-x[1])[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    print(f"{100*v/tot:5.1f}% L{ln:>4} inst={inst[ln]:.2e} {src.get(ln,'').strip()[:90]}")
