"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle.

Tolerances: relative L2 <= 1e-5 (north star, fp32 GPU vs double oracle on the
same fp32 inputs) unless a reference test pins a looser bound (brute-force
oracle 3e-3); peak locations exact.  Each test names the reference test or
BASELINE config it follows.
"""
import os

import numpy as np
import pytest

import paper_2006_13188_b200 as X

pytestmark = pytest.mark.gpu
ROT, SCALE = 0, 1
TOL = 1e-5


def ofilter(orc, F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def pfilter(F):
    return X.FreqFilter2(F.group, F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                         F.r_min, F.r_domain)


def xfield(kind, p):
    return X.XformField.rotation(p) if kind == ROT else X.XformField.scaling(p)


def full_decomp(orc, filt, R, n_radii=24, n_angles=64):
    return orc.decompose_rotation2(filt, R, R, n_angles, n_radii, n_angles, R)


# ------------------------------------------------------ reference KATs on GPU

@pytest.mark.parametrize("mode", [0, 1])
def test_rotation_matches_oracle_fast_path(orc, mode):  # test_engine2d.cpp:140-153
    rng = orc.Rng(55)
    n, R = 24, 6
    F = full_decomp(orc, rng.random_smooth_filter(R), R)
    H = rng.random_field(n, n, False)
    T = rng.random_rotation_field(n, n)
    ref = (orc.xcorr_fast if mode == 0 else orc.xconv_fast)(H, ROT, T, F)[0]
    fn = X.xcorr_fast if mode == 0 else X.xconv_fast
    r = fn(H, X.XformField.rotation(T), pfilter(F))
    assert r.standard_ops == F.n_components()
    assert orc.rel_l2(r.output, ref) < TOL
    assert orc.rel_l2(r.output, orc.spectral_oracle(mode, H, ROT, T, F)) < TOL


@pytest.mark.parametrize("mode", [0, 1])
def test_scale_matches_oracle(orc, mode):  # test_engine_scale.cpp:121-134
    rng = orc.Rng(73)
    n, R = 20, 6
    F = orc.decompose_scale2(rng.annular_filter(R), R, R, 8, 48, 32, 1.0, R)
    H = rng.random_field(n, n, False)
    T = rng.random_scale_field(n, n)
    ref = (orc.xcorr_fast if mode == 0 else orc.xconv_fast)(H, SCALE, T, F)[0]
    fn = X.xcorr_fast if mode == 0 else X.xconv_fast
    r = fn(H, X.XformField.scaling(T), pfilter(F))
    assert orc.rel_l2(r.output, ref) < TOL


def test_rotation_fast_matches_brute(orc):  # test_engine2d.cpp:123-138
    rng = orc.Rng(54)
    n, R = 24, 6
    F = full_decomp(orc, rng.random_smooth_filter(R), R)
    PF = pfilter(F)
    for _ in range(3):
        H = rng.random_field(n, n, False)
        T = rng.random_rotation_field(n, n)
        assert orc.rel_l2(X.xcorr_fast(H, X.XformField.rotation(T), PF).output,
                          orc.xcorr_brute(H, ROT, T, F)) < 3e-3
        assert orc.rel_l2(X.xconv_fast(H, X.XformField.rotation(T), PF).output,
                          orc.xconv_brute(H, ROT, T, F)) < 3e-3


def test_single_component_plan(orc):  # test_engine2d.cpp:176-194
    rng = orc.Rng(57)
    n, R = 16, 5
    F = full_decomp(orc, rng.random_smooth_filter(R), R, 16, 32)
    H = rng.random_field(n, n, True)
    T = rng.random_rotation_field(n, n)
    r = X.xcorr_fast(H, X.XformField.rotation(T), pfilter(F), X.XConvPlan(components=[2]))
    assert r.standard_ops == 1
    F2 = orc.render_component(F, F.index_of(2), 2 * R + 1, 2 * R + 1, R, R)
    ref = orc.filter2_fft(H, F2, R, R, True) * np.exp(2j * T)
    assert orc.rel_l2(r.output, ref) < TOL


def test_periodic_matches_oracle_and_is_equivariant(orc):  # test_engine2d.cpp:196-219
    rng = orc.Rng(58)
    n, R = 16, 4
    F = full_decomp(orc, rng.random_smooth_filter(R), R, 12, 32)
    H = rng.random_field(n, n, True)
    T = rng.random_rotation_field(n, n)
    plan = X.XConvPlan(periodic=True)
    base = X.xcorr_fast(H, X.XformField.rotation(T), pfilter(F), plan).output
    assert orc.rel_l2(base, orc.xcorr_fast(H, ROT, T, F, periodic=True)[0]) < TOL
    sh = X.xcorr_fast(np.roll(H, (3, 5), (0, 1)), X.XformField.rotation(np.roll(T, (3, 5), (0, 1))),
                      pfilter(F), plan).output
    assert np.max(np.abs(np.roll(base, (3, 5), (0, 1)) - sh)) < 1e-5 * np.max(np.abs(base))
    conv = X.xconv_fast(H, X.XformField.rotation(T), pfilter(F), plan).output
    assert orc.rel_l2(conv, orc.xconv_fast(H, ROT, T, F, periodic=True)[0]) < TOL


def test_op_count_and_validation(orc):  # test_engine2d.cpp:221-235, 285-299
    rng = orc.Rng(59)
    n, R = 12, 4
    filt = rng.random_smooth_filter(R)
    H = rng.random_field(n, n, True)
    T = X.XformField.rotation(rng.random_rotation_field(n, n))
    for K in (0, 2, 4, 8):
        F = X.decompose_rotation2(filt, R, R, K, 12, 32, R)
        assert X.xcorr_fast(H, T, F).standard_ops == 2 * (K // 2) + 1
        assert X.xconv_fast(H, T, F).standard_ops == 2 * (K // 2) + 1
    F = X.decompose_rotation2(filt, R, R, 8, 12, 32, R)
    with pytest.raises(ValueError, match="signal and transformation field dims differ"):
        X.xcorr_fast(H, X.XformField.rotation(np.zeros((8, 8))), F)
    with pytest.raises(ValueError, match="transformation/filter group mismatch"):
        X.xcorr_fast(H, X.XformField.scaling(np.ones((n, n))), F)
    with pytest.raises(ValueError, match="plan retains a component the filter lacks"):
        X.xcorr_fast(H, T, F, X.XConvPlan(components=[99]))


def test_scale_guard_band_names_pixel(orc):  # test_engine_scale.cpp:161-178
    rng = orc.Rng(76)
    n, R = 8, 5
    F = orc.decompose_scale2(rng.annular_filter(R), R, R, 4, 48, 32, 1.0, R)
    H = rng.random_field(n, n, True)
    s = np.ones((n, n))
    s[3, 5] = 10.0
    with pytest.raises(ValueError) as ei:
        X.xcorr_fast(H, X.XformField.scaling(s), pfilter(F))
    msg = str(ei.value)
    with pytest.raises(ValueError) as eo:
        orc.xcorr_fast(H, SCALE, s, F)
    assert "guard band" in msg and "(5,3)" in msg and msg == str(eo.value)


def test_real_in_real_out(orc):  # test_engine2d.cpp:237-248
    rng = orc.Rng(60)
    n, R = 18, 5
    F = pfilter(full_decomp(orc, rng.random_smooth_filter(R), R, 16, 32))
    H = rng.random_field(n, n, False)
    T = X.XformField.rotation(rng.random_rotation_field(n, n))
    for fn in (X.xcorr_fast, X.xconv_fast):
        out = fn(H, T, F).output
        assert np.max(np.abs(out.imag)) < 1e-6 * np.max(np.abs(out))


# ------------------------------------------------------------------ smooth

def test_smooth_matches_oracle(orc):  # test_smooth.cpp:108-137
    rng = orc.Rng(91)
    n, R = 32, 6
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    g = np.exp(-(x * x + y * y) / (2 * 1.8 ** 2))
    g[x * x + y * y > R * R] = 0
    F = orc.decompose_scale2(g, R, R, 62, 64, 16, 0.5, R, R + 3.0)
    H = np.full((n, n), 0.7)
    S = rng.random_scale_field(n, n)
    out = X.smooth_adaptive(H, X.XformField.scaling(S), pfilter(F))
    assert np.max(np.abs(out.output - 0.7)) < 1e-5
    assert out.standard_ops == 2 * F.n_components()
    Hs = orc.gaussian_blur(rng.random_field(n, n, False).real, 2.0)
    ref, ops, cl = orc.smooth_adaptive(Hs, SCALE, S, F)
    got = X.smooth_adaptive(Hs, X.XformField.scaling(S), pfilter(F))
    assert orc.rel_l2(got.output, ref) < TOL and got.clamped_pixels == cl
    bad = X.smooth_adaptive(Hs, X.XformField.scaling(S), pfilter(F), normalize_signal=False)
    ref_bad = orc.smooth_adaptive(Hs, SCALE, S, F, False)[0]
    assert orc.rel_l2(bad.output, ref_bad) < TOL


def test_smooth_zero_integral_rejected(orc):  # test_smooth.cpp:174-187
    R = 5
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    f = x * np.exp(-(x * x + y * y) / 8.0)
    F = X.decompose_rotation2(f, R, R, 8, 2 * R, 32, R)
    with pytest.raises(ValueError, match="normalization undefined: filter has zero integral"):
        X.smooth_adaptive(np.ones((16, 16)), X.XformField.rotation(np.zeros((16, 16))), F)


# ------------------------------------------------------- BASELINE configs

def _cfg_parity(orc, w, n_check_pix=0):
    """GPU vs oracle on one (reduced-size) config image."""
    OF = ofilter(orc, w.filt)
    H = w.signal[0].astype(np.float64)
    if w.mode in ("xcorr", "xconv"):
        fn = X.xcorr_fast if w.mode == "xcorr" else X.xconv_fast
        got = fn(w.signal[0], xfield(w.kind, w.param[0]), w.filt).output
        ofn = orc.xcorr_fast if w.mode == "xcorr" else orc.xconv_fast
        ref = ofn(H, w.kind, w.param[0].astype(np.float64), OF)[0]
        return orc.rel_l2(got, ref)
    if w.mode == "smooth":
        got = X.smooth_adaptive(w.signal[0], xfield(w.kind, w.param[0]), w.filt).output
        ref = orc.smooth_adaptive(H, w.kind, w.param[0].astype(np.float64), OF)[0]
        return orc.rel_l2(got, ref)
    raise AssertionError(w.mode)


def test_config1_full_size(orc):
    from paper_2006_13188_b200 import workloads as WL
    assert _cfg_parity(orc, WL.config1()) < TOL


def test_config2_reduced(orc):
    from paper_2006_13188_b200 import workloads as WL
    assert _cfg_parity(orc, WL.config2(n=192)) < TOL


def test_config4_reduced(orc):
    from paper_2006_13188_b200 import workloads as WL
    assert _cfg_parity(orc, WL.config4(n=160)) < TOL


def test_config5_reduced(orc):
    from paper_2006_13188_b200 import workloads as WL
    assert _cfg_parity(orc, WL.config5(n=160, batch=1)) < TOL


def test_config3_reduced_anglemax_and_peaks(orc):
    from paper_2006_13188_b200 import workloads as WL
    w = WL.config3(n=320, n_templates=2)
    OF = ofilter(orc, w.filt)
    score, arg = X.anglemax(w.signal[0], w.filt, 360)
    # oracle: per-band G_k via single-component xcorr_fast with zero angle
    H = w.signal[0].astype(np.float64)
    zero = np.zeros_like(H)
    G = np.stack([orc.xcorr_fast(H, ROT, zero, OF, components=[int(k)])[0] for k in OF.ks])
    oscore, oarg = orc.anglemax(G, OF.ks, 360)
    assert orc.rel_l2(score, oscore) < TOL
    # argmax: the oracle's value at the GPU's angle attains the oracle max
    s = np.arange(360)
    at = np.abs(np.einsum("kyx,kyx->yx", G,
                          np.exp(-2j * np.pi * np.asarray(OF.ks)[:, None, None] * arg[None] / 360)))
    assert np.all(at >= oscore * (1 - 1e-5) - 1e-9)
    pk = X.find_peaks(score.astype(np.float64), 32.0, 0.5)
    opk = orc.find_peaks(oscore, 32.0, 0.5)
    assert [(p.x, p.y) for p in pk[:2]] == [(p[0], p[1]) for p in opk[:2]]
    for (cx, cy, _), p in zip(sorted(w.meta["truth"]), sorted(pk[:2], key=lambda q: q.x)):
        assert abs(p.x - cx) <= 2 and abs(p.y - cy) <= 2


@pytest.mark.parametrize("cfg,mode", [(1, 0), (5, 0), (2, 1)])
def test_full_size_sampled_pixels(orc, cfg, mode):
    """Full BASELINE sizes (one image): GPU vs the spectral oracle at sampled pixels
    (the spectral oracle equals the FFT path to 1e-8, test_engine2d.cpp:140-153)."""
    from paper_2006_13188_b200 import workloads as WL
    w = {1: WL.config1, 2: WL.config2, 5: lambda: WL.config5(batch=1)}[cfg]()
    fn = X.xcorr_fast if mode == 0 else X.xconv_fast
    got = fn(w.signal[0], X.XformField.rotation(w.param[0]), w.filt).output
    r = np.random.default_rng(7)
    h, wd = got.shape
    ys = np.concatenate([r.integers(0, h, 48), [0, h - 1, 0, h - 1]])
    xs = np.concatenate([r.integers(0, wd, 48), [0, 0, wd - 1, wd - 1]])
    ref = orc.spectral_oracle_at(mode, w.signal[0], ROT, w.param[0], ofilter(orc, w.filt), ys, xs)
    assert orc.rel_l2(got[ys, xs], ref) < TOL


# ---------------------------------------------------------- dtypes & layout

def test_dtypes_batch_and_colmajor(orc):
    rng = orc.Rng(100)
    n, R = 40, 6
    F = full_decomp(orc, rng.random_smooth_filter(R), R)
    PF = pfilter(F)
    H = np.stack([rng.random_field(n, n + 3, True) for _ in range(3)])
    T = np.stack([rng.random_rotation_field(n, n + 3) for _ in range(3)])
    got = X.xcorr_fast(H, X.XformField.rotation(T), PF).output  # complex128 batch
    for b in range(3):
        ref = orc.xcorr_fast(H[b], ROT, T[b], F)[0]
        assert orc.rel_l2(got[b], ref) < TOL
    got32 = X.xcorr_fast(H.astype(np.complex64), X.XformField.rotation(T.astype(np.float32)), PF)
    assert got32.output.dtype == np.complex64
    assert orc.rel_l2(got32.output[1], got[1]) < TOL
    # column-major (Eigen) storage through the C ABI, as the C++ shim passes it
    import ctypes as C
    from paper_2006_13188_b200 import _native as N
    Hc = np.asfortranarray(H[0])
    Tc = np.asfortranarray(T[0])
    out = np.zeros((n + 3, n), np.complex128, order="F")
    d = N.ImageDesc(n + 3, n, 1, N.XC_C128, N.XC_F64, N.XC_C128, N.XC_COL_MAJOR, N.XC_HOST, 0,
                    N.XC_ROTATION2)
    ctx = N.context()
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, PF.handle(), 0, C.byref(d), Hc.ctypes.data, Tc.ctypes.data,
                           None, 0, 0, out.ctypes.data, C.byref(st)), ctx.handle)
    assert orc.rel_l2(out, orc.xcorr_fast(H[0], ROT, T[0], F)[0]) < TOL


@pytest.mark.parametrize("shape", [(1, 1), (1, 9), (7, 1), (3, 5), (13, 2)])
def test_tiny_and_ragged_images(orc, shape):
    rng = orc.Rng(101)
    R = 6
    F = full_decomp(orc, rng.random_smooth_filter(R), R)
    h, w = shape
    H = rng.random_field(w, h, True)
    T = rng.random_rotation_field(w, h)
    for mode, fn, ofn in ((0, X.xcorr_fast, orc.xcorr_fast), (1, X.xconv_fast, orc.xconv_fast)):
        got = fn(H, X.XformField.rotation(T), pfilter(F)).output
        assert orc.rel_l2(got, ofn(H, ROT, T, F)[0]) < TOL
        gotp = fn(H, X.XformField.rotation(T), pfilter(F), X.XConvPlan(periodic=True)).output
        assert orc.rel_l2(gotp, ofn(H, ROT, T, F, periodic=True)[0]) < TOL


# --------------------------------------------- fast-path coverage (pad table)

@pytest.mark.parametrize("n_angles,m_max", [(360, 4), (360, 8), (100, 4)])
@pytest.mark.parametrize("real_filter", [False, True])
def test_anglemax_fft_and_generic(orc, n_angles, m_max, real_filter):
    """360 angles with |m| <= KH runs the FFT evaluation; other n the Horner one.
    A real filter on a real signal takes the Hermitian half-band path
    (G_{-k} = conj G_k: only k >= 0 transformed) where it applies."""
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(5)
    f = WL.angular_filter(9, 4.0, m_max, r)
    if real_filter:
        f = f.real + 0.0j
    F = X.decompose_rotation2(f, 9, 9, 2 * m_max, 18, 4 * m_max + 4, 9.0)
    H = r.standard_normal((70, 90)).astype(np.float32)
    score, arg = X.anglemax(H, F, n_angles)
    OF = ofilter(orc, F)
    G = np.stack([orc.xcorr_fast(H.astype(np.float64), ROT, np.zeros(H.shape), OF,
                                 components=[int(k)])[0] for k in OF.ks])
    oscore, oarg = orc.anglemax(G, OF.ks, n_angles)
    assert orc.rel_l2(score, oscore) < TOL
    at = np.abs(np.einsum("kyx,kyx->yx", G, np.exp(
        -2j * np.pi * np.asarray(OF.ks)[:, None, None] * arg[None] / n_angles)))
    assert np.all(at >= oscore * (1 - 1e-5) - 1e-9)


@pytest.mark.parametrize("n", [256, 480])
def test_fast_scatter_and_smooth_sizes(orc, n):
    """Pads 288 / 512 are fast-table lengths: S1/S2 fast kernels (rotation
    scatter, scale smoothing) against the oracle."""
    from paper_2006_13188_b200 import workloads as WL
    w = WL.config2(n=n)
    assert _cfg_parity(orc, w) < TOL
    w4 = WL.config4(n=n)
    assert _cfg_parity(orc, w4) < TOL
    # scale-group gather (fast I1/I2 + conj(dc) H)
    H = w4.signal[0]
    S = w4.param[0]
    got = X.xcorr_fast(H, X.XformField.scaling(S), w4.filt).output
    ref = orc.xcorr_fast(H.astype(np.float64), SCALE, S.astype(np.float64), ofilter(orc, w4.filt))[0]
    assert orc.rel_l2(got, ref) < TOL


def test_host_pipeline_batch_matches_device_path(orc):
    """Host-memory batches (two-slot H2D/compute/D2H pipeline) equal per-image calls."""
    from paper_2006_13188_b200 import workloads as WL
    w = WL.config1()
    r = np.random.default_rng(9)
    B = 5
    sig = r.uniform(0, 1, (B, 256, 256)).astype(np.float32)
    th = r.uniform(0, 2 * np.pi, (B, 256, 256)).astype(np.float32)
    batch = X.xcorr_fast(sig, X.XformField.rotation(th), w.filt).output
    for b in (0, 3, 4):
        one = X.xcorr_fast(sig[b], X.XformField.rotation(th[b]), w.filt).output
        assert np.array_equal(batch[b], one)


# ------------------------------------------------- pair-engine geometry edges

def _direct_at(orc, F, H, theta, ys, xs, periodic):
    """out(p) = sum_k e^{i k theta(p)} sum_u conj(F_k(u)) H(p + u) (fft.hpp:74-77,
    engine.hpp:312-317) evaluated directly in double at the sampled pixels."""
    R = int(np.ceil(F.r_max))
    side = 2 * R + 1
    comps = np.stack([orc.render_component(F, ci, side, side, R, R) for ci in range(len(F.ks))])
    h, w = H.shape
    d = np.arange(-R, R + 1)
    out = np.zeros(len(ys), np.complex128)
    for i, (y, x) in enumerate(zip(ys, xs)):
        yy, xx = y + d, x + d
        if periodic:
            patch = H[np.ix_(yy % h, xx % w)].astype(np.float64)
        else:
            patch = np.zeros((side, side))
            vy, vx = (yy >= 0) & (yy < h), (xx >= 0) & (xx < w)
            patch[np.ix_(vy, vx)] = H[np.ix_(yy[vy], xx[vx])]
        g = np.einsum("kab,ab->k", np.conj(comps), patch)
        out[i] = np.sum(np.exp(1j * np.asarray(F.ks) * float(theta[y, x])) * g)
    return out


@pytest.mark.parametrize("h,w,periodic", [(4101, 4000, False), (4000, 4101, False),
                                          (4275, 4275, True)])
def test_pair_engine_geometry_edges(orc, h, w, periodic):
    """Transform length 4320 (the pair-engine kernels) with an odd height, a
    different row length, and the periodic wrap with an odd crop offset R=15."""
    from paper_2006_13188_b200 import workloads as WL
    wk = WL.config1(n=64)
    Fo = ofilter(orc, wk.filt)
    # the direct sum agrees with the oracle's FFT path on a small image first
    r = np.random.default_rng(11)
    Hs = r.uniform(0, 1, (40, 37)).astype(np.float32)
    Ts = r.uniform(0, 2 * np.pi, (40, 37)).astype(np.float32)
    ref_s = orc.xcorr_fast(Hs.astype(np.float64), ROT, Ts.astype(np.float64), Fo)[0]
    yy, xx = np.array([0, 5, 39, 20]), np.array([0, 36, 3, 18])
    assert orc.rel_l2(_direct_at(orc, Fo, Hs, Ts, yy, xx, False), ref_s[yy, xx]) < 1e-10
    H = r.uniform(0, 1, (h, w)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
    res = X.xcorr_fast(H, X.XformField.rotation(T), wk.filt, X.XConvPlan(periodic=periodic))
    got = res.output
    ys = np.concatenate([r.integers(0, h, 40), [0, h - 1, 0, h - 1, h // 2]])
    xs = np.concatenate([r.integers(0, w, 40), [0, 0, w - 1, w - 1, 1]])
    ref = _direct_at(orc, Fo, H, T, ys, xs, periodic)
    assert orc.rel_l2(got[ys, xs], ref) < TOL


@pytest.mark.parametrize("images_per_i1", ["1", "2"])
def test_pair_engine_image_groups(orc, images_per_i1):
    """Batches on the 4320 pad run I1 on two images per launch (one staged
    filter spectrum shared): every image of an odd batch (a group of two plus
    a single) must equal its single-image result bit for bit, through host and
    device memory, and match the direct oracle at sampled pixels."""
    import subprocess
    import sys
    if os.environ.get("XCB_I1_IMAGES", "1") != images_per_i1:
        # the setting is read once per process: run this case in a child
        env = dict(os.environ, XCB_I1_IMAGES=images_per_i1)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__ +
                            f"::test_pair_engine_image_groups[{images_per_i1}]"], env=env,
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        return
    import torch
    from paper_2006_13188_b200 import workloads as WL
    wk = WL.config1(n=64)
    r = np.random.default_rng(12)
    n = 4100
    H = r.uniform(0, 1, (3, n, n)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (3, n, n)).astype(np.float32)
    batch = X.xcorr_fast(H, X.XformField.rotation(T), wk.filt).output
    for b in range(3):
        one = X.xcorr_fast(H[b], X.XformField.rotation(T[b]), wk.filt).output
        assert np.array_equal(batch[b], one)
    import ctypes as C
    from paper_2006_13188_b200 import _native as N
    hs, ts = torch.from_numpy(H).cuda(), torch.from_numpy(T).cuda()
    out = torch.empty((3, n, n), dtype=torch.complex64, device="cuda")
    d = N.ImageDesc(n, n, 3, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1,
                    N.XC_ROTATION2)
    ctx = N.context()
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, wk.filt.handle(), 0, C.byref(d), C.c_void_p(hs.data_ptr()),
                           C.c_void_p(ts.data_ptr()), None, 0, 0, C.c_void_p(out.data_ptr()),
                           C.byref(st)), ctx.handle)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), batch)
    ys, xs = r.integers(0, n, 24), r.integers(0, n, 24)
    ref = _direct_at(orc, ofilter(orc, wk.filt), H[1], T[1], ys, xs, False)
    assert orc.rel_l2(batch[1][ys, xs], ref) < TOL


def _bands_at(orc, F, H, ys, xs):
    """G_k(p) = sum_u conj(F_k(u)) H(p + u) (fft.hpp:74-77, zero padding) per band at
    the sampled pixels, in double; shape (bands, samples)."""
    R = int(np.ceil(F.r_max))
    side = 2 * R + 1
    comps = np.stack([orc.render_component(F, ci, side, side, R, R) for ci in range(len(F.ks))])
    h, w = H.shape
    d = np.arange(-R, R + 1)
    G = np.zeros((len(F.ks), len(ys)), np.complex128)
    for i, (y, x) in enumerate(zip(ys, xs)):
        yy, xx = y + d, x + d
        patch = np.zeros((side, side))
        vy, vx = (yy >= 0) & (yy < h), (xx >= 0) & (xx < w)
        patch[np.ix_(vy, vx)] = H[np.ix_(yy[vy], xx[vx])]
        G[:, i] = np.einsum("kab,ab->k", np.conj(comps), patch)
    return G


def test_config3_full_size_anglemax(orc):
    """BASELINE config 3 at full size (4096^2, 33 bands, 360 angles): score and
    argmax at sampled pixels (including the pasted templates' centres) against
    the direct per-band correlation + the oracle's angle max, and the top-3 NMS
    peaks at the templates (vote_filter.hpp:107-134)."""
    from paper_2006_13188_b200 import workloads as WL
    w = WL.config3()
    OF = ofilter(orc, w.filt)
    score, arg = X.anglemax(w.signal[0], w.filt, 360)
    truth = w.meta["truth"]
    r = np.random.default_rng(31)
    n = score.shape[0]
    ys = np.concatenate([r.integers(0, n, 30), [int(round(cy)) for _, cy, _ in truth], [0, n - 1]])
    xs = np.concatenate([r.integers(0, n, 30), [int(round(cx)) for cx, _, _ in truth], [n - 1, 0]])
    G = _bands_at(orc, OF, w.signal[0].astype(np.float64), ys, xs)
    oscore, oarg = orc.anglemax(G[:, None, :], OF.ks, 360)
    oscore = oscore[0]
    assert orc.rel_l2(score[ys, xs], oscore) < TOL
    at = np.abs(np.sum(G * np.exp(-2j * np.pi * np.asarray(OF.ks)[:, None] * arg[ys, xs][None] / 360),
                       axis=0))
    assert np.all(at >= oscore * (1 - 1e-5) - 1e-9)
    pk = X.find_peaks(score.astype(np.float64), 32.0, 0.5)
    assert len(pk) >= 3
    for (cx, cy, _), p in zip(sorted(truth), sorted(pk[:3], key=lambda q: q.x)):
        assert abs(p.x - cx) <= 2 and abs(p.y - cy) <= 2


def _scatter_at(orc, F, x, phi, ys, xs, periodic=False):
    """Scatter (xconv) at sampled pixels, direct in double: out(p) =
    sum_u sum_k F_k(u) e^{-i k phi(p-u)} x(p-u) (fft.hpp:74-77 convolution,
    engine.hpp:353-358 premultiply), zero padding or periodic wrap."""
    R = int(np.ceil(F.r_max))
    side = 2 * R + 1
    comps = np.stack([orc.render_component(F, ci, side, side, R, R) for ci in range(len(F.ks))])
    ks = np.asarray(F.ks, np.float64)
    h, w = x.shape
    d = np.arange(-R, R + 1)
    out = np.zeros(len(ys), np.complex128)
    for i, (y, xx0) in enumerate(zip(ys, xs)):
        qy, qx = y - d, xx0 - d  # q = p - u for u = (d_y, d_x)
        if periodic:
            qy, qx = qy % h, qx % w
        vy, vx = (qy >= 0) & (qy < h), (qx >= 0) & (qx < w)
        xv = np.zeros((side, side))
        ph = np.zeros((side, side))
        xv[np.ix_(vy, vx)] = x[np.ix_(qy[vy], qx[vx])]
        ph[np.ix_(vy, vx)] = phi[np.ix_(qy[vy], qx[vx])]
        steer = np.exp(-1j * ks[:, None, None] * ph[None])
        out[i] = np.sum(comps * steer * xv[None])
    return out


def test_config4_full_size_smoothing(orc):
    """BASELINE config 4 at full size (2048^2, 13 log-radial bands, s in [1, 8]):
    smooth_adaptive (engine.hpp:385-419) through the pair-engine S1/S2 kernels
    (pad 2160) against a direct scatter of H/s^2 and 1/s^2 at sampled pixels."""
    from paper_2006_13188_b200 import workloads as WL
    w = WL.config4()
    OF = ofilter(orc, w.filt)
    H = w.signal[0].astype(np.float64)
    S = w.param[0].astype(np.float64)
    got = X.smooth_adaptive(w.signal[0], X.XformField.scaling(w.param[0]), w.filt)
    assert got.clamped_pixels == 0
    r = np.random.default_rng(41)
    n = H.shape[0]
    ys = np.concatenate([r.integers(0, n, 24), [0, n - 1, 0, n - 1]])
    xs = np.concatenate([r.integers(0, n, 24), [0, 0, n - 1, n - 1]])
    phi = OF.omega() * np.log(S)
    wgt = 1.0 / (S * S)
    dc = orc.inner_dc_value(OF)
    num = _scatter_at(orc, OF, H * wgt, phi, ys, xs) + dc * (H * wgt)[ys, xs]
    den = _scatter_at(orc, OF, wgt, phi, ys, xs) + dc * wgt[ys, xs]
    ref = (num / den).real
    assert orc.rel_l2(got.output[ys, xs], ref) < TOL


@pytest.mark.parametrize("real_filter", [False, True])
def test_scatter_hermitian_half_band(orc, real_filter):
    """xconv_fast of a real signal with a real filter (F_{-k} = conj F_k) takes the
    Hermitian half-band path on the pair engine (bands k >= 0, out = 2 Re); a
    complex filter takes the full path.  Both against the spectral oracle at
    sampled pixels (pad 1152)."""
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(17)
    f = WL.angular_filter(16, 8.0, 8, r)
    if real_filter:
        f = f.real + 0.0j
    F = X.decompose_rotation2(f, 16, 16, 16, 32, 34, 16.0)
    n = 1024
    H = r.uniform(0, 1, (n, n)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (n, n)).astype(np.float32)
    got = X.xconv_fast(H, X.XformField.rotation(T), F).output
    if real_filter:
        assert np.max(np.abs(got.imag)) == 0.0
    ys = np.concatenate([r.integers(0, n, 40), [0, n - 1, 0, n - 1]])
    xs = np.concatenate([r.integers(0, n, 40), [0, 0, n - 1, n - 1]])
    ref = orc.spectral_oracle_at(1, H, ROT, T, ofilter(orc, F), ys, xs)
    assert orc.rel_l2(got[ys, xs], ref) < TOL


@pytest.mark.parametrize("h,w,periodic,real_filter", [(1101, 1000, False, False),
                                                      (1101, 1101, True, False),
                                                      (1101, 1101, True, True)])
def test_scatter_pair_engine_geometry_edges(orc, h, w, periodic, real_filter):
    """Scatter on the pair engine at pad 1152 with an odd height, a row length on
    another plan (1024), and the periodic wrap (odd crop offset R = 17), in the
    full and the Hermitian half-band modes, against a direct scatter."""
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(23)
    f = WL.angular_filter(17, 7.0, 6, r)
    if real_filter:
        f = f.real + 0.0j
    F = X.decompose_rotation2(f, 17, 17, 12, 24, 28, 16.5)
    H = r.uniform(0, 1, (h, w)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
    got = X.xconv_fast(H, X.XformField.rotation(T), F, X.XConvPlan(periodic=periodic)).output
    ys = np.concatenate([r.integers(0, h, 30), [0, h - 1, 0, h - 1]])
    xs = np.concatenate([r.integers(0, w, 30), [0, 0, w - 1, w - 1]])
    ref = _scatter_at(orc, ofilter(orc, F), H.astype(np.float64), T.astype(np.float64), ys, xs,
                      periodic)
    assert orc.rel_l2(got[ys, xs], ref) < TOL


@pytest.mark.parametrize("n,batch,real_filter", [(1024, 1, True), (1024, 1, False),
                                                  (4101, 2, True)])
def test_gather_hermitian_half_band(orc, n, batch, real_filter):
    """xcorr_fast of real signals with a real filter (F_{-k} = conj F_k) takes the
    Hermitian half-band gather (I1 over bands k >= 0, I2 with the k = 0 band at
    weight 1/2 and out = 2 Re) on the pair engine: pad 1152 (single image) and
    pad 4320 (two images per I1 launch).  A complex filter takes the full path.
    Against the spectral oracle at sampled pixels."""
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(29)
    f = WL.angular_filter(15, 6.0, 6, r)
    if real_filter:
        f = f.real + 0.0j
    F = X.decompose_rotation2(f, 15, 15, 8, 30, 32, 15.0)
    H = r.uniform(0, 1, (batch, n, n)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (batch, n, n)).astype(np.float32)
    got = X.xcorr_fast(H if batch > 1 else H[0], X.XformField.rotation(T if batch > 1 else T[0]),
                       F).output.reshape(batch, n, n)
    if real_filter:
        assert np.max(np.abs(got.imag)) == 0.0
    OF = ofilter(orc, F)
    for b in range(batch):
        ys = np.concatenate([r.integers(0, n, 30), [0, n - 1, 0, n - 1]])
        xs = np.concatenate([r.integers(0, n, 30), [0, 0, n - 1, n - 1]])
        ref = orc.spectral_oracle_at(0, H[b], ROT, T[b], OF, ys, xs)
        assert orc.rel_l2(got[b][ys, xs], ref) < TOL


def test_dual_i1_i2_batches_match_single_images(orc):
    """XCB_DUAL=1 (opt-in): gather batches on the 4320 pad run I1 of image i and
    I2 of image i-1 in one launch (k_dual_ilv).  Every image must equal its
    single-image result bit for bit (host and device memory paths)."""
    import subprocess
    import sys
    if os.environ.get("XCB_DUAL") != "1":
        env = dict(os.environ, XCB_DUAL="1")
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__ +
                            "::test_dual_i1_i2_batches_match_single_images"], env=env,
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        return
    from paper_2006_13188_b200 import workloads as WL
    wk = WL.config1(n=64)
    r = np.random.default_rng(31)
    n = 4100
    H = r.uniform(0, 1, (3, n, n)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (3, n, n)).astype(np.float32)
    batch = X.xcorr_fast(H, X.XformField.rotation(T), wk.filt).output
    for b in range(3):
        one = X.xcorr_fast(H[b], X.XformField.rotation(T[b]), wk.filt).output
        assert np.array_equal(batch[b], one)
    ys, xs = r.integers(0, n, 16), r.integers(0, n, 16)
    ref = _direct_at(orc, ofilter(orc, wk.filt), H[2], T[2], ys, xs, False)
    assert orc.rel_l2(batch[2][ys, xs], ref) < TOL


@pytest.mark.parametrize("n,K", [(2048, 16), (2048, 4)])
def test_i1_tail_split_pad_2160(orc, n, K):
    """Pad 2160 runs 1,080 column pairs at two CTAs per SM: 3 full waves and a
    partial one of 192 pairs.  With 17 bands the partial wave is split into 3
    band chunks per column pair (k_pair.cu tail_split); with 5 bands it is not.
    Both against the spectral oracle at sampled pixels."""
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(41)
    f = WL.angular_filter(15, 6.0, K // 2, r)
    F = X.decompose_rotation2(f, 15, 15, K, 30, 2 * K + 2, 15.0)
    H = r.uniform(0, 1, (n, n)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (n, n)).astype(np.float32)
    res = X.xcorr_fast(H, X.XformField.rotation(T), F)
    assert res.standard_ops == 2 * (K // 2) + 1
    ys = np.concatenate([r.integers(0, n, 40), [0, n - 1, 0, n - 1]])
    xs = np.concatenate([r.integers(0, n, 40), [0, 0, n - 1, n - 1]])
    ref = orc.spectral_oracle_at(0, H, ROT, T, ofilter(orc, F), ys, xs)
    assert orc.rel_l2(res.output[ys, xs], ref) < TOL
