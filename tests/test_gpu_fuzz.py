"""Randomized parity sweep: xcorr_fast / xconv_fast / smooth_adaptive on the GPU
against the CPU oracle over random image shapes (odd, ragged, thin), both
groups, random band limits and component subsets, periodic mode, complex and
real signals, fp32 / fp64 inputs and Eigen column-major layout.  Every case
must be within relative L2 1e-5 and report the reference's op count.

XCB_FUZZ_CASES=N widens the sweep (the default keeps it to seconds)."""
import os

import numpy as np
import pytest

import paper_2006_13188_b200 as X

pytestmark = pytest.mark.gpu
TOL = 1e-5
N_CASES = int(os.environ.get("XCB_FUZZ_CASES", "24"))


def _case(orc, seed):
    r = np.random.default_rng([seed, 2006])
    kind = int(r.integers(0, 2))  # 0 rotation2, 1 scale2
    R = int(r.integers(2, 9))
    h = int(r.integers(1, 90))
    w = int(r.integers(1, 90))
    if r.random() < 0.2:  # thin images
        h = int(r.integers(1, 4))
    mode = ["xcorr", "xconv", "smooth"][int(r.integers(0, 3))]
    periodic = mode != "smooth" and r.random() < 0.25 and h > 2 * R and w > 2 * R
    cplx = mode != "smooth" and r.random() < 0.5
    f64 = r.random() < 0.3
    colmajor = r.random() < 0.3
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    filt = np.zeros_like(x)
    for _ in range(4):
        bx, by = r.uniform(-R / 2, R / 2, 2)
        filt += r.uniform(-1, 1) * np.exp(-((x - bx) ** 2 + (y - by) ** 2) / (2 * r.uniform(1, 2) ** 2))
    filt = filt * np.exp(-(x * x + y * y) / (2 * (0.45 * R) ** 2))
    if mode == "smooth":  # a smoothing kernel: positive, so the denominator stays away from 0
        filt = np.abs(filt) + 0.05 * np.exp(-(x * x + y * y) / (2 * (0.45 * R) ** 2))
    elif r.random() < 0.5:
        filt = filt + 1j * r.uniform(-0.3, 0.3) * np.roll(filt, 1, axis=1)
    if kind == 0:
        K = int(r.integers(2, 2 * R + 1))
        na = max(16, 2 * K + 2)
        na += na % 2
        F = X.decompose_rotation2(filt, R, R, K, 2 * R, na, float(R))
    else:
        K = int(r.integers(2, 10))
        F = X.decompose_scale2(filt, R, R, K, max(K + 2, 12), 16, 1.0, float(R))
    ks = list(F.ks)
    comps = []
    if mode != "smooth" and r.random() < 0.3:
        comps = sorted(r.choice(ks, size=int(r.integers(1, len(ks) + 1)), replace=False).tolist())
    H = r.uniform(0, 1, (h, w)) + (1j * r.uniform(-1, 1, (h, w)) if cplx else 0)
    if kind == 0:
        P = r.uniform(-np.pi, np.pi, (h, w))
    else:  # inside the guard band [r_min / r_top, r_top / r_min]
        P = np.exp(r.uniform(np.log(0.6), np.log(1.6), (h, w)))
    dt = np.complex128 if cplx else np.float64
    if not f64:
        dt = np.complex64 if cplx else np.float32
    Hc = H.astype(dt)
    Pc = P.astype(np.float64 if f64 else np.float32)
    return dict(kind=kind, mode=mode, periodic=periodic, colmajor=colmajor, F=F, comps=comps,
                H=Hc, P=Pc, desc=f"seed {seed}: {mode} {'scale' if kind else 'rot'} {h}x{w} R={R} "
                                   f"K={K} bands={len(ks)} sub={comps} periodic={periodic} "
                                   f"cplx={cplx} f64={f64} colmajor={colmajor}")


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_case_matches_oracle(orc, seed):
    c = _case(orc, seed)
    F = c["F"]
    OF = orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max, F.r_min,
                    F.r_domain)
    H, P = c["H"], c["P"]
    Href, Pref = H.astype(np.complex128), P.astype(np.float64)
    T = X.XformField.rotation(P) if c["kind"] == 0 else X.XformField.scaling(P)
    if c["mode"] == "smooth":
        got = X.smooth_adaptive(H, T, F)
        ref, ops, clamped = orc.smooth_adaptive(Href, c["kind"], Pref, OF, True)
        assert got.standard_ops == ops, c["desc"]
        out = got.output
    else:
        plan = X.XConvPlan(components=c["comps"], periodic=c["periodic"])
        fn = X.xcorr_fast if c["mode"] == "xcorr" else X.xconv_fast
        ofn = orc.xcorr_fast if c["mode"] == "xcorr" else orc.xconv_fast
        if c["colmajor"]:
            # the C ABI's Eigen column-major path through the same call: transpose in,
            # transpose out (the library solves the transposed problem)
            from paper_2006_13188_b200 import _native as N
            import ctypes as C
            Ht = np.asfortranarray(H)
            Pt = np.asfortranarray(P)
            wide = H.dtype in (np.float64, np.complex128)
            outc = np.zeros(H.shape, np.complex128 if wide else np.complex64, order="F")
            sdt = {np.dtype(np.float32): N.XC_F32, np.dtype(np.float64): N.XC_F64,
                   np.dtype(np.complex64): N.XC_C64, np.dtype(np.complex128): N.XC_C128}[H.dtype]
            d = N.ImageDesc(H.shape[0], H.shape[1], 1, sdt,
                            N.XC_F64 if P.dtype == np.float64 else N.XC_F32,
                            N.XC_C128 if wide else N.XC_C64, N.XC_COL_MAJOR, N.XC_HOST, 1,
                            c["kind"])
            comp = np.ascontiguousarray(np.asarray(c["comps"], np.int32))
            st = N.Stats()
            ctx = N.context(0)
            N.check(N.lib().xc_run(ctx.handle, F.handle(), 0 if c["mode"] == "xcorr" else 1,
                                   C.byref(d), Ht.ctypes.data, Pt.ctypes.data,
                                   comp.ctypes.data_as(C.POINTER(C.c_int)) if len(comp) else None,
                                   len(comp), N.XC_FLAG_PERIODIC if c["periodic"] else 0,
                                   outc.ctypes.data, C.byref(st)), ctx.handle)
            out, got_ops = outc, st.standard_ops
        else:
            got = fn(H, T, F, plan)
            out, got_ops = got.output, got.standard_ops
        ref, ops, _ = ofn(Href, c["kind"], Pref, OF, components=c["comps"] or None,
                          periodic=c["periodic"])
        assert got_ops == ops, c["desc"]
    err = orc.rel_l2(out, ref)
    assert err < TOL, f"{c['desc']}: rel_l2 {err:.3e}"
