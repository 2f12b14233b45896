timeout 900 python -m pytest tests/test_gpu_cpair.py -x -q -rA 2>&1 | tail -30 > gpurun_out/s5c8_cpair_tests.log; echo rc=$? >> gpurun_out/s5c8_cpair_tests.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c8_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c8_gpu_tests.log
python - > gpurun_out/s5c8_modes.txt 2>&1 <<'PY'
import ctypes as C, numpy as np, time
import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N, workloads as WL
r = np.random.default_rng(1)
F = X.decompose_rotation2(WL.angular_filter(10, 4.0, 8, r), 10, 10, 16, 20, 36, 10.0)
ctx = N.context(0)
for n in (64, 250, 500, 1000, 2000, 3400, 4000):
    H = r.uniform(0, 1, (n, n)).astype(np.float32); T = r.uniform(0, 6.28, (n, n)).astype(np.float32)
    out = np.zeros(H.shape, np.complex64)
    d = N.ImageDesc(n, n, 1, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_HOST, 1, 0)
    st = N.Stats()
    for i in range(3):
        N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), 1, C.byref(d), H.ctypes.data, T.ctypes.data, None, 0, 0, out.ctypes.data, C.byref(st)), ctx.handle)
    print(n, "pad", st.pad_h, st.pad_w, "mode", st.band_mode, "bands_run", st.bands_run, "gpu s", round(st.seconds_fft * 1e3, 3), "ms")
PY
