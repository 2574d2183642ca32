"""Summarise an `ncu --page source --csv` SASS dump: top instructions and
per-opcode totals of executed warp instructions and stall samples."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(float(r[ix["Instructions Executed"]] or 0) for r in data)
samp = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total warp instructions executed {tot:.3e}, stall samples {samp:.0f}")
op = collections.Counter()
ops = collections.Counter()
for r in data:
    o = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if o.startswith("@"):
        o = r[ix["Source"]].split()[1]
    o = o.split(".")[0]
    op[o] += float(r[ix["Instructions Executed"]] or 0)
    ops[o] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
print("opcode            executed%   stall%")
for k, v in op.most_common(25):
    print(f"{k:16s} {100*v/tot:8.2f} {100*ops[k]/max(samp,1):8.2f}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("\nhottest instructions by stall samples:")
for r in sorted(data, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
    print(f'{r[ix["Address"]]:>6s} {float(r[ix["Warp Stall Sampling (All Samples)"]] or 0):7.0f} '
          f'{float(r[ix["Instructions Executed"]] or 0):11.0f} {r[ix["Avg. Threads Executed"]]:>6s}  {r[ix["Source"]][:70]}')
