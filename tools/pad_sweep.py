"""Per-stage device times of xconv / xcorr (device-resident inputs) over image
sizes around the pair-plan pads, to compare a fast-plan pad with the next
pair-plan pad (XCB_PAD_PAIR=0/1)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N, workloads as WL

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sizes = [int(a) for a in sys.argv[2:]] or [900, 1000, 1900, 2000, 3400, 3900, 4000]
r = np.random.default_rng(1)
F = X.decompose_rotation2(WL.angular_filter(10, 4.0, 8, r), 10, 10, 16, 20, 36, 10.0)
ctx = N.context(0)
dev = torch.device("cuda", 0)
for n in sizes:
    H = torch.from_numpy(r.uniform(0, 1, (n, n)).astype(np.float32)).to(dev)
    T = torch.from_numpy(r.uniform(0, 6.28, (n, n)).astype(np.float32)).to(dev)
    out = torch.empty((n, n), dtype=torch.complex64, device=dev)
    torch.cuda.synchronize()
    d = N.ImageDesc(n, n, 1, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1, 0)
    st = N.Stats()

    def call():
        N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), mode, C.byref(d), H.data_ptr(),
                               T.data_ptr(), None, 0, 0, out.data_ptr(), C.byref(st)), ctx.handle)
    for _ in range(3):
        call()
    ctx.profile(enable=True, reset=True)
    for _ in range(10):
        call()
    prof = ctx.profile(enable=False, reset=True)
    tot = sum(v[0] for v in prof.values()) / 10
    print(n, "pad", st.pad_h, "mode", st.band_mode, "total %.3f ms" % tot,
          {k: round(v[0] / 10, 3) for k, v in prof.items()}, flush=True)
    ctx.trim()
