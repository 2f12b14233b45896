"""Key metrics and top stall reasons per kernel from an ncu --page raw --csv export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled")
         and h.endswith("per_issue_active.ratio")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("----", d.get("Kernel Name", "")[:100])
    for w in want:
        print(f"  {w:60s} {d.get(w)}")
    st = sorted(((float(d[s]) if d[s] not in ("", "n/a") else 0, s) for s in stall), reverse=True)[:8]
    print("  stalls/issue: " + ", ".join(
        f"{s.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
        f"={v:.2f}" for v, s in st))
