set -x
for v in 1 2; do for pr in 0 1 2 3 4 5 6; do
XCB_TC_VARIANT=$v XCB_TC_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:anglemax_tc -c 2 --csv python tools/profile_case.py anglemax 3 2>/dev/null | grep anglemax_tc | tail -1 | awk -F'","' -v v=$v -v p=$pr '{print "v" v " probe" p " " $NF}' >> gpurun_out/r2c13_probes.txt
done; done
