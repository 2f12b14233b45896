"""Device-resident timing of every BASELINE config through the public API
(timed without profiling; the per-stage CUDA-event profile comes from a
separate pass).  Prints one JSON line per config."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_13188_b200 import _native as N  # noqa: E402
from paper_2006_13188_b200 import workloads as WL  # noqa: E402


def run(cfg, reps=3):
    w = {5: lambda: WL.config5(batch=2)}.get(cfg, WL.CONFIGS[cfg])()
    dev = torch.device("cuda", 0)
    ctx = N.context(0)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    B, H, W = w.signal.shape
    sig = torch.from_numpy(w.signal).to(dev)
    fh = w.filt.handle()
    st = N.Stats()
    if w.mode in ("xcorr", "xconv"):
        par = torch.from_numpy(w.param).to(dev)
        out = torch.empty((B, H, W), dtype=torch.complex64, device=dev)
        d = N.ImageDesc(H, W, B, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1,
                        int(w.filt.group))
        mode = 0 if w.mode == "xcorr" else 1

        def call():
            N.check(N.lib().xc_run(ctx.handle, fh, mode, C.byref(d), C.c_void_p(sig.data_ptr()),
                                   C.c_void_p(par.data_ptr()), None, 0, 0,
                                   C.c_void_p(out.data_ptr()), C.byref(st)), ctx.handle)
    elif w.mode == "smooth":
        par = torch.from_numpy(w.param).to(dev)
        out = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        d = N.ImageDesc(H, W, B, N.XC_F32, N.XC_F32, N.XC_F32, N.XC_ROW_MAJOR, N.XC_DEVICE, 1,
                        int(w.filt.group))

        def call():
            N.check(N.lib().xc_smooth(ctx.handle, fh, C.byref(d), C.c_void_p(sig.data_ptr()),
                                      C.c_void_p(par.data_ptr()), 1, C.c_void_p(out.data_ptr()),
                                      C.byref(st)), ctx.handle)
    else:
        out = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        arg = torch.empty((B, H, W), dtype=torch.int32, device=dev)
        d = N.ImageDesc(H, W, B, N.XC_F32, N.XC_F32, N.XC_F32, N.XC_ROW_MAJOR, N.XC_DEVICE, 0, 0)

        def call():
            N.check(N.lib().xc_anglemax(ctx.handle, fh, C.byref(d), C.c_void_p(sig.data_ptr()),
                                        None, 0, 360, C.c_void_p(out.data_ptr()),
                                        C.cast(C.c_void_p(arg.data_ptr()), C.POINTER(C.c_int)),
                                        C.byref(st)), ctx.handle)
    call()
    torch.cuda.synchronize()
    # timed calls without the per-stage events (small configs take more reps)
    reps_t = reps if B * H * W >= 1 << 22 else 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps_t):
        call()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps_t
    # stage breakdown from a separate profiled pass
    ctx.profile(enable=True, reset=True)
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
    prof = ctx.profile(enable=False, reset=True)
    units = w.units()
    print(json.dumps({"config": cfg, "workload": w.name, "ms_per_call": ms,
                      "Mpix_bands_per_s": units / ms / 1e3, "pad": [st.pad_h, st.pad_w],
                      "standard_ops": st.standard_ops, "launches_per_call": st.gpu_launches,
                      "stages_ms": {k: v[0] / reps for k, v in prof.items()}}), flush=True)


def run_peaks_detect(reps=5):
    """find_peaks on the GPU over config 3's 4096^2
    score map (NMS radius 32, threshold 0.5; the host sorts), and detect_pattern
    (gradient + 33-band scatter + NMS) on a 2048^2 scene, through the public API
    with host buffers."""
    import paper_2006_13188_b200 as X
    w = WL.config3()
    score, _ = X.anglemax(w.signal[0], w.filt, 360)
    dev = torch.device("cuda", 0)
    s = torch.from_numpy(score).to(dev)
    X.find_peaks(s, 32.0, 0.5, gpu=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        pk = X.find_peaks(s, 32.0, 0.5, gpu=True)
    dt = (time.perf_counter() - t0) / reps
    print(json.dumps({"config": "A10", "workload": "find_peaks_device 4096^2 (config 3 score)",
                      "ms_per_call": dt * 1e3, "Mpix_per_s": score.size / dt / 1e6,
                      "peaks": len(pk)}), flush=True)
    rng = np.random.default_rng(5)
    R = 16
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    pat = (np.exp(-((x - 5) ** 2 + (y + 3) ** 2) / 18.0) -
           0.8 * np.exp(-((x + 6) ** 2 + (y - 4) ** 2) / 12.0)) * np.exp(-(x * x + y * y) / 200.0)
    img = rng.normal(0, 0.02, (2048, 2048))
    for cx, cy, a in ((400.5, 700.0, 0.4), (1500.0, 300.0, 2.1), (1200.0, 1600.0, -1.0)):
        WL.paste_rotated(img, pat, cx, cy, a)
    img = img.astype(np.float32)
    vf = X.build_optimal_filter(pat, R, R, float(R))
    det = X.detect_pattern(img, vf, 32)
    t0 = time.perf_counter()
    for _ in range(reps):
        det = X.detect_pattern(img, vf, 32)
    dt = (time.perf_counter() - t0) / reps
    print(json.dumps({"config": "F1", "workload": "detect_pattern 2048^2, K=32 (33 bands), eps 16",
                      "ms_per_call": dt * 1e3,
                      "Mpix_bands_per_s": img.size * det.standard_ops / dt / 1e6,
                      "standard_ops": det.standard_ops,
                      "top_peaks": [(p.x, p.y) for p in det.peaks[:3]]}), flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["1", "2", "3", "4", "5", "extra"]):
        if c == "extra":
            run_peaks_detect()
        else:
            run(int(c))
