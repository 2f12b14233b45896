"""Print SASS context (with the dominant stall reasons) around given addresses
of an ncu --page source --csv --print-source sass export.
usage: ncu_ctx.py export.csv ADDR[,ADDR...] [before] [after]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:  # first kernel section only (later sections repeat the header)
    if r and r[0] == "Address":
        break
    if len(r) == len(hdr):
        data.append(r)
stalls = [h for h in hdr if h.startswith("stall_")]
before = int(sys.argv[3]) if len(sys.argv) > 3 else 12
after = int(sys.argv[4]) if len(sys.argv) > 4 else 4
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
pos = {r[0]: i for i, r in enumerate(data)}
for a in sys.argv[2].split(","):
    i = next(v for k, v in pos.items() if k.endswith(a))  # full address or its hex suffix
    print(f"---- {a}")
    for r in data[max(0, i - before):i + after + 1]:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
        why = " ".join(f"{h}={v / max(s, 1):.0%}" for v, h in top if v)
        print(f"{r[0][-5:]} {s / tot:6.2%} {r[ix['Source']][:60]:60s} {why}")
