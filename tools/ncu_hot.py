"""Summarise an ncu --page source --csv --print-source sass export: the SASS
instructions with the most warp-stall samples, and stall totals by opcode."""
import csv
import collections
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
samp = [(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r) for r in data
        if len(r) == len(hdr) and r[ix["Warp Stall Sampling (All Samples)"]].isdigit()]
tot = sum(s for s, _ in samp)
print("total samples", tot)
by_op = collections.Counter()
ex_op = collections.Counter()
for s, r in samp:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    by_op[op] += s
    ex_op[op] += int(r[ix["Instructions Executed"]] or 0)
print("stall samples by opcode (share) / warp-instructions executed")
for op, s in by_op.most_common(25):
    print(f"  {op:10s} {s/tot:6.1%}  {ex_op[op]:>12d}")
print("top instructions")
for s, r in sorted(samp, key=lambda x: -x[0])[:top]:
    print(f"  {s/tot:6.2%} {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:70]}")

# per stall reason: the instructions collecting most of it
if len(sys.argv) > 3:
    for reason in sys.argv[3].split(","):
        col = ix.get("stall_" + reason)
        if col is None:
            continue
        seen = set()
        lst = []
        for s, r in samp:
            if r[ix["Address"]] in seen:
                continue
            seen.add(r[ix["Address"]])
            v = int(r[col] or 0)
            if v:
                lst.append((v, r))
        tot_r = sum(v for v, _ in lst)
        print(f"stall_{reason}: {tot_r} samples")
        for v, r in sorted(lst, key=lambda x: -x[0])[:12]:
            print(f"  {v/tot_r:6.1%} {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:70]}")
