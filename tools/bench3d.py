"""Timing of the 3D rotation pipeline through the public API:
xcorr_fast_3d / xconv_fast_3d on an n^3 volume, filter radius R, degree
limit K (sum (2l+1)^2 bands).  Prints one JSON line per mode with the device
time (CUDA events inside xc_run3), the end-to-end call time (host buffers,
H2D/D2H included) and the oracle's CPU time per band on a sample of degrees.

  python tools/bench3d.py [--n 64] [--R 4] [--K 4] [--reps 5] [--cpu-degrees 0,1]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13188_b200 as X  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (CPU baseline leg only)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--R", type=int, default=4)
ap.add_argument("--K", type=int, default=4)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--cpu-degrees", default="0,1")
a = ap.parse_args()

rng = np.random.default_rng(3)
n, R, K = a.n, a.R, a.K
y, x, z = np.mgrid[-R:R + 1, -R:R + 1, -R:R + 1]
vol = np.exp(-(x * x + y * y + z * z) / (2 * (0.4 * R) ** 2)) * (1 + 0.5 * x / R + 0.3 * y * z / R ** 2)
G = X.decompose_rotation3(vol, R, R, R, K, 2 * R, float(R), max(12, 2 * K + 2), max(12, 2 * K + 2))
H = rng.random((n, n, n))
q = rng.normal(size=(n, n, n, 4))
q /= np.linalg.norm(q, axis=-1, keepdims=True)
T = X.rotation3d(q)
bands = sum((2 * l + 1) ** 2 for l in range(K + 1))
F = orc.Filter3(G.K, G.n_radii, G.r_max, G.coeffs)
cpu_deg = [int(s) for s in a.cpu_degrees.split(",")]
cpu_bands = sum((2 * l + 1) ** 2 for l in cpu_deg)
for mode, fn in (("xcorr_3d", X.xcorr_fast_3d), ("xconv_3d", X.xconv_fast_3d)):
    fn(H, T, G)  # warm-up: filter spectra cache, plans, buffers
    dev, e2e = [], []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        r = fn(H, T, G)
        e2e.append(time.perf_counter() - t0)
        dev.append(r.seconds["fft"])
    t0 = time.perf_counter()
    orc.xfast3(0 if mode == "xcorr_3d" else 1, H, q, F, degrees=cpu_deg)
    cpu_s = time.perf_counter() - t0
    units = n ** 3 * bands
    print(json.dumps({
        "workload": mode, "n": n, "R": R, "K": K, "bands": bands, "standard_ops": r.standard_ops,
        "gpu_launches": r.gpu_launches,
        "device_ms": 1e3 * float(np.median(dev)), "e2e_ms": 1e3 * float(np.median(e2e)),
        "Mvoxel_bands_per_s": units / float(np.median(dev)) / 1e6,
        "e2e_Mvoxel_bands_per_s": units / float(np.median(e2e)) / 1e6,
        "cpu_baseline": {"Mvoxel_bands_per_s": n ** 3 * cpu_bands / cpu_s / 1e6, "cores": 1,
                         "kind": "port",
                         "sample": f"degrees {cpu_deg} ({cpu_bands} bands), {cpu_s:.1f} s"}}))
