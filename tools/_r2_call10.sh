set -x
for pr in 0 1; do XCB_TC_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:anglemax_tc -c 2 --csv python tools/profile_case.py anglemax 3 > gpurun_out/r2c10_probe$pr.csv 2>&1; done
timeout 300 ncu --set full --clock-control none -k regex:"anglemax_tc" -c 1 -o /tmp/am_tc python tools/profile_case.py anglemax 3 > /dev/null 2>&1
ncu -i /tmp/am_tc.ncu-rep --page raw --csv > gpurun_out/r2c10_tc_raw.csv 2>/dev/null
