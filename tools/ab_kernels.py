"""A/B kernel timing at locked (base) clocks: for each library build in
paper_2006_13188_b200/lib/ab/*.so (or the names given), run
tools/profile_case.py under ncu --clock-control base and print the mean
duration per kernel.  Power capping makes free-running clocks move by a few
percent between runs; this isolates code changes.  Never a bench number.

  python tools/ab_kernels.py [--case "xcorr 5 1"] [--regex ilv] [NAME ...]
"""
import argparse
import collections
import csv
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--case", default="xcorr 5 1")
ap.add_argument("--regex", default="ilv")
ap.add_argument("names", nargs="*")
a = ap.parse_args()
libdir = os.path.join(ROOT, "paper_2006_13188_b200", "lib", "ab")
names = a.names or sorted(os.path.basename(p)[:-3] for p in glob.glob(os.path.join(libdir, "*.so")))
res = {}
for n in names:
    out = f"/tmp/ab_{n}.csv"
    env = dict(os.environ, XCB_LIB_OVERRIDE=os.path.join(libdir, n + ".so"))
    cmd = ["ncu", "--clock-control", "base", "--metrics", "gpu__time_duration.sum", "-k",
           f"regex:{a.regex}", "--csv", "--log-file", out, sys.executable,
           os.path.join(ROOT, "tools", "profile_case.py"), *a.case.split()]
    subprocess.run(cmd, env=env, check=True, capture_output=True)
    rows = [r for r in csv.reader(l for l in open(out) if l.startswith('"'))]
    ix = {h: i for i, h in enumerate(rows[0])}
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        unit = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[ix["Metric Unit"]]]
        agg[r[ix["Kernel Name"]].split("(")[0].split("<")[0].split("::")[-1]].append(
            float(r[ix["Metric Value"]].replace(",", "")) * unit)
    res[n] = {k: sum(v) / len(v) for k, v in agg.items()}
kern = sorted({k for v in res.values() for k in v})
print("kernel".ljust(32) + "".join(n[:14].rjust(15) for n in names))
for k in kern:
    print(k[:32].ljust(32) + "".join(
        (f"{res[n][k]:13.1f}us" if k in res[n] else "-".rjust(15)) for n in names))
