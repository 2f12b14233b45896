"""Host-buffer call breakdown (xc_stats seconds_*) for the small configs."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N, workloads as WL

for cfg in (2, 1):
    w = WL.CONFIGS[cfg]()
    H, Wd = w.signal.shape[1:]
    hs = torch.from_numpy(w.signal[0]).pin_memory()
    hp = torch.from_numpy(w.param[0]).pin_memory()
    ho = torch.empty((H, Wd), dtype=torch.complex64).pin_memory()
    ctx = N.context(0)
    d = N.ImageDesc(H, Wd, 1, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_HOST, 1, 0)
    st = N.Stats()
    mode = 1 if w.mode == "xconv" else 0
    def call():
        N.check(N.lib().xc_run(ctx.handle, w.filt.handle(ctx), mode, C.byref(d), hs.data_ptr(),
                               hp.data_ptr(), None, 0, 0, ho.data_ptr(), C.byref(st)), ctx.handle)
    for _ in range(5):
        call()
    t0 = time.perf_counter()
    n = 50
    for _ in range(n):
        call()
    dt = (time.perf_counter() - t0) / n
    print(f"cfg{cfg}: wall {dt*1e3:.3f} ms/call; stats total {st.seconds_total*1e3:.3f} fft {st.seconds_fft*1e3:.3f} "
          f"h2d {st.seconds_h2d*1e3:.3f} d2h {st.seconds_d2h*1e3:.3f} ms; launches {st.gpu_launches}")
    # raw copy times for the same buffers
    ds = torch.empty((H, Wd), dtype=torch.float32, device="cuda")
    do = torch.empty((H, Wd), dtype=torch.complex64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        ds.copy_(hs, non_blocking=True); ds.copy_(hp, non_blocking=True); ho.copy_(do, non_blocking=True)
        torch.cuda.synchronize()
    print(f"   raw pinned copies (2 in + 1 out): {(time.perf_counter()-t0)/n*1e3:.3f} ms")
