set -x
for v in 0 1 2; do
XCB_TC_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_anglemax_tc.py -x -q > gpurun_out/r2c11_tc_v$v.log 2>&1; echo rc=$? >> gpurun_out/r2c11_tc_v$v.log
for pr in 0 1; do XCB_TC_VARIANT=$v XCB_TC_PROBE=$pr timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:anglemax_tc -c 2 --csv python tools/profile_case.py anglemax 3 2>/dev/null | grep anglemax_tc > gpurun_out/r2c11_v${v}_probe$pr.csv; done
done
