"""Markdown share table from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0]
    ns = float(r[ix["Metric Value"]].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0, r[ix["Block Size"]], r[ix["Grid Size"]]])
    a[0] += 1
    a[1] += ns
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | total ms | share | block | grid |")
print("|---|---|---|---|---|---|")
for name, (n, ns, bs, gs) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{name}` | {n} | {ns / 1e6:.2f} | {ns / tot:.1%} | {bs} | {gs} |")
