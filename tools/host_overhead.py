"""Per-call host overhead of xc_run with device-resident buffers (no CUDA graph):
synchronous calls, and XC_FLAG_ASYNC calls issued back to back (one sync at the
end), against the kernels' device time."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N, workloads as WL

dev = torch.device("cuda", 0)
for cfg in (1, 2):
    w = WL.CONFIGS[cfg]()
    H, Wd = w.signal.shape[1:]
    ds = torch.from_numpy(w.signal[0]).to(dev)
    dp = torch.from_numpy(w.param[0]).to(dev)
    do = torch.empty((H, Wd), dtype=torch.complex64, device=dev)
    torch.cuda.synchronize()
    ctx = N.context(0)
    d = N.ImageDesc(H, Wd, 1, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1, 0)
    st = N.Stats()
    mode = 1 if w.mode == "xconv" else 0
    fh = w.filt.handle(ctx)

    def call(flags):
        N.check(N.lib().xc_run(ctx.handle, fh, mode, C.byref(d), ds.data_ptr(), dp.data_ptr(),
                               None, 0, flags, do.data_ptr(), C.byref(st)), ctx.handle)
    for _ in range(5):
        call(0)
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        call(0)
    t_sync = (time.perf_counter() - t0) / n
    for _ in range(5):
        call(N.XC_FLAG_ASYNC)
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        call(N.XC_FLAG_ASYNC)
    t_issue = (time.perf_counter() - t0) / n
    ctx.synchronize()
    t_async = (time.perf_counter() - t0) / n
    print(f"cfg{cfg}: sync call {t_sync*1e6:.1f} us; async issue {t_issue*1e6:.1f} us/call, "
          f"async throughput {t_async*1e6:.1f} us/call; kernels (stats of the last sync call) "
          f"{st.seconds_fft*1e6:.1f} us; launches {st.gpu_launches}")
