"""Summarise an `ncu --page source --csv` dump: top SASS lines by stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot = sum(float(r[idx['Warp Stall Sampling (All Samples)']] or 0) for r in data)
ins = sum(float(r[idx['Instructions Executed']] or 0) for r in data)
print(f'total samples {tot:.0f}, warp instructions executed {ins:.3e}')
data.sort(key=lambda r: -float(r[idx['Warp Stall Sampling (All Samples)']] or 0))
for r in data[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    s = float(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    print(f"{100*s/tot:5.1f}%  {r[idx['Address']]:>6}  {r[idx['Source']][:70]:70s} exec={r[idx['Instructions Executed']]}")
