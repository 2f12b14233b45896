"""Per-launch kernel statistics from ncu --set full captures, keyed
"cfg<N>:<stage>" as bench.py names its stages, into profiles/ncu_kernel_stats.json
(bench.py reads it for roofline.traffic and the issue roofline).

  python tools/ncu_stats.py OUT.json CFG:REPORT.ncu-rep [CFG:REPORT ...]

Each report is exported with `ncu -i REPORT --page raw --csv`; several launches
of one stage are averaged; the smoothing finish (max + divide kernels) sums.
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

STAGES = [  # kernel-name pattern -> bench stage
    (r"k_cols_inv_corr", "I1_cols_inv_corr"), (r"k_rows_inv_steer", "I2_rows_inv_steer"),
    (r"k_rows_inv_planes", "I2_rows_inv_planes"), (r"k_rows_fwd_premul", "S1_rows_fwd_premul"),
    (r"k_cols_fwd_mac", "S2_cols_fwd_mac_inv"), (r"k_rows_inv_out", "S4_rows_inv_out"),
    (r"k_rows_fwd_ilv", "F1_rows_fwd"), (r"k_cols_fwd_ilv", "F2_cols_fwd"),
    (r"k_anglemax", "anglemax"), (r"k_smooth", "smooth_finish"), (r"k_prep", "prep"),
    (r"k_absmax", "absmax"),
]
SUMMED = {"smooth_finish"}  # several kernels per launch of the stage


def stage_of(name):
    for pat, st in STAGES:
        if re.search(pat, name):
            return st
    return None


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    scale = {h: UNIT.get(u, 1.0) for h, u in zip(hdr, units)}
    return [{h: (num(v) * scale[h] if h in NUMERIC else v) for h, v in zip(hdr, r)}
            for r in rows[2:]]


# to bytes / ns / plain numbers
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
        "second": 1e9, "s": 1e9}
NUMERIC = {"dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
           "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"}


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return 0.0


def main():
    out_path = sys.argv[1]
    res = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for arg in sys.argv[2:]:
        cfg, rep = arg.split(":", 1)
        if not os.path.exists(rep):
            print(f"skip {rep}: missing", file=sys.stderr)
            continue
        acc = collections.defaultdict(lambda: collections.defaultdict(float))
        cnt = collections.Counter()
        for d in rows_of(rep):
            st = stage_of(d.get("Kernel Name", ""))
            if st is None:
                continue
            a = acc[st]
            a["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            a["warp_instructions"] += d.get("smsp__inst_executed.sum", 0)
            a["duration_ns"] += d.get("gpu__time_duration.sum", 0)
            a["issue_active_pct"] += d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0)
            cnt[st] += 1
        for st, a in acc.items():
            n = 1 if st in SUMMED else cnt[st]
            k = 1.0 / n
            res[f"cfg{cfg}:{st}"] = {
                "dram_bytes": a["dram_bytes"] * k, "warp_instructions": a["warp_instructions"] * k,
                "ncu_duration_ms": a["duration_ns"] * k * 1e-6,
                "issue_active_pct": a["issue_active_pct"] / cnt[st],
                "launches_averaged": n, "source": os.path.basename(rep)}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)
    print(json.dumps(res, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
