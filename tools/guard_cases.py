"""Out-of-bounds check driver (the GPU pool has no compute-sanitizer):
runs every pipeline once on cuda:0 and saves the outputs to an .npz; with
XCB_GUARD=<bytes> in the environment every context buffer is guarded and
poisoned (api.cu guard_bytes), and the guard zones are checked at the end.
tests/test_gpu_guards.py runs it twice (guarded and plain) and requires
bit-identical outputs and untouched guards.

  [XCB_GUARD=65536] python tools/guard_cases.py OUT.npz
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13188_b200 as X  # noqa: E402
from paper_2006_13188_b200 import _native as N  # noqa: E402
from paper_2006_13188_b200 import workloads as WL  # noqa: E402


def cases():
    out = {}
    rng = np.random.default_rng(5)
    # pair engine at every table length: 1152 (scatter), 2160 (smoothing), 4320 (gather)
    w2 = WL.config2()
    T2 = X.XformField.rotation(w2.param[0])
    out["cfg2_xconv"] = X.xconv_fast(w2.signal[0], T2, w2.filt).output
    out["cfg2_xcorr"] = X.xcorr_fast(w2.signal[0], T2, w2.filt).output
    w4 = WL.config4()
    out["cfg4_smooth"] = X.smooth_adaptive(w4.signal[0], X.XformField.scaling(w4.param[0]),
                                           w4.filt).output
    w5 = WL.config5(batch=1)
    out["cfg5_xcorr"] = X.xcorr_fast(w5.signal[0], X.XformField.rotation(w5.param[0]),
                                     w5.filt).output
    sub = X.XConvPlan(components=[int(k) for k in w5.filt.ks[::3]])
    out["cfg5_xconv_subset"] = X.xconv_fast(w5.signal[0], X.XformField.rotation(w5.param[0]),
                                            w5.filt, sub).output
    # angle max (planes + the Hermitian DFT kernel) on a reduced config 3
    w3 = WL.config3(n=1024, n_templates=2)
    am = X.anglemax(w3.signal[0], w3.filt, 360)
    out["cfg3_score"], out["cfg3_argmax"] = np.asarray(am[0]), np.asarray(am[1])
    # generic / fast kernels: config 1, ragged and tiny images, periodic mode
    w1 = WL.config1()
    T1 = X.XformField.rotation(w1.param[0])
    out["cfg1_xcorr"] = X.xcorr_fast(w1.signal[0], T1, w1.filt).output
    for h, w in [(97, 61), (13, 2), (1, 9), (7, 1)]:
        H = rng.random((h, w)).astype(np.float32)
        th = (rng.random((h, w)) * 2 * np.pi).astype(np.float32)
        T = X.XformField.rotation(th)
        out[f"rag{h}x{w}_xcorr"] = X.xcorr_fast(H, T, w1.filt).output
        out[f"rag{h}x{w}_xconv"] = X.xconv_fast(H, T, w1.filt).output
    # the session-5 pair plans (rows / columns on different lengths: 768 x 1280,
    # 2880 x 576, 3072 + 4096 with the fast and the split paired S2), the angle
    # max at one of them, and halo tiles beyond 4320
    for h, w in [(740, 1250), (2860, 560), (3050, 200), (150, 4070)]:
        H = rng.random((h, w)).astype(np.float32)
        T = X.XformField.rotation((rng.random((h, w)) * 2 * np.pi).astype(np.float32))
        out[f"len{h}x{w}_xcorr"] = X.xcorr_fast(H, T, w1.filt).output
        out[f"len{h}x{w}_xconv"] = X.xconv_fast(H, T, w1.filt).output
    Hn = rng.standard_normal((1500, 700)).astype(np.float32)
    am2 = X.anglemax(Hn, w1.filt, 360)
    out["len1500x700_score"], out["len1500x700_argmax"] = np.asarray(am2[0]), np.asarray(am2[1])
    for h, w in [(4400, 130), (120, 4500)]:
        H = rng.random((h, w)).astype(np.float32)
        T = X.XformField.rotation((rng.random((h, w)) * 2 * np.pi).astype(np.float32))
        out[f"tile{h}x{w}_xcorr"] = X.xcorr_fast(H, T, w1.filt).output
        out[f"tile{h}x{w}_xconv"] = X.xconv_fast(H, T, w1.filt).output
    per = X.XConvPlan(periodic=True)
    out["cfg1_periodic"] = X.xcorr_fast(w1.signal[0], T1, w1.filt, per).output
    # device decomposition + pattern detection
    R = 8  # test_detect.cpp:11-31 style pattern: Gaussian bumps under an envelope
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    pat = np.exp(-((x - 2.5) ** 2 + (y + 1.0) ** 2) / 3.0) - 0.8 * np.exp(
        -((x + 2.0) ** 2 + (y - 2.0) ** 2) / 2.0)
    pat *= np.exp(-(x * x + y * y) / (2 * (0.38 * R) ** 2))
    vf = X.build_optimal_filter(pat, float(R), float(R), float(R))
    img = np.zeros((80, 96))
    img[20:37, 30:47] += pat
    img[50:67, 60:77] += pat[::-1].T
    out["detect_response"] = np.asarray(X.detect_pattern(img, vf, 16).response)
    Fd = X.decompose_rotation2(w2.filter_image, *w2.decomp[1], device=True)
    out["decomp_device"] = np.asarray(Fd.comps)
    # 3D
    n3 = 12
    vol = rng.random((7, 7, 7)).astype(np.complex128)
    G = X.decompose_rotation3(vol, 3, 3, 3, 2, 6, 3.0)
    q = rng.standard_normal((n3, n3, n3, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    H3 = rng.random((n3, n3, n3))
    out["xcorr3"] = X.xcorr_fast_3d(H3, X.rotation3d(q), G).output
    out["xconv3"] = X.xconv_fast_3d(H3, X.rotation3d(q), G).output
    return out


if __name__ == "__main__":
    res = cases()
    np.savez(sys.argv[1], **{k: np.asarray(v) for k, v in res.items()})
    guard = N.lib().xc_debug_guard_bytes()
    bad, name = N.context(0).check_guards() if guard else (0, "")
    print(json.dumps({"guard_bytes": guard, "bad_guards": bad, "first_bad": name,
                      "cases": len(res),
                      "nonfinite": sorted(k for k, v in res.items()
                                          if not np.all(np.isfinite(np.asarray(v))))}))
