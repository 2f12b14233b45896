"""GPU parity for the scatter's conjugate band pairs (xconv_fast of a real
signal, engine.hpp:331-373): S1 transforms the bands k >= 0 only, S2 feeds
each column FFT into two sums (F^_k and the spectrum of conj f_{-k}), S4 writes
a + conj(b).  Every case is compared with the CPU oracle (full image, relative
L2 <= 1e-5) at a pad with a pair plan (1152 or 2160); the selections that do
not qualify (asymmetric band subsets, complex signals) must take the full path
and give the same answers.
"""
import os

import numpy as np
import pytest

import paper_2006_13188_b200 as X

pytestmark = pytest.mark.gpu
ROT, SCALE = 0, 1
TOL = 1e-5
NT = min(16, os.cpu_count() or 1)


def ofilter(orc, F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def _rot_case(seed, h, w, m_max=6, R=12):
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(seed)
    f = WL.angular_filter(R, R / 2.5, m_max, r)  # complex coefficients: F_{-k} != conj F_k
    F = X.decompose_rotation2(f, R, R, 2 * m_max, 24, 4 * m_max + 4, float(R))  # bands -m_max..m_max
    H = r.uniform(0, 1, (h, w)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
    return r, F, H, T


@pytest.mark.parametrize("h,w", [(1024, 1024), (1001, 1100), (1100, 2100)])
def test_cpair_full_image_matches_oracle(orc, h, w):
    """Square, odd-height and mixed-plan (rows 2160, columns 1152) geometries."""
    r, F, H, T = _rot_case(101, h, w)
    res = X.xconv_fast(H, X.XformField.rotation(T), F)
    assert res.standard_ops == len(F.ks)
    ref = orc.xconv_fast(H.astype(np.float64), ROT, T.astype(np.float64), ofilter(orc, F),
                         nthreads=NT)[0]
    assert orc.rel_l2(res.output, ref) < TOL
    # no symmetry is imposed on the output: the imaginary part is significant
    assert np.linalg.norm(ref.imag) > 0.1 * np.linalg.norm(ref.real)


@pytest.mark.parametrize("comps", [[3, 1, 0, -1, -3], [5, -5], [2, 0, -1], [4, 3, 2], [0]])
def test_cpair_band_subsets(orc, comps):
    """Symmetric subsets (non-unit band steps, no k = 0 band) take the paired
    path; asymmetric ones, one-sided ones and a lone band the full path."""
    r, F, H, T = _rot_case(102, 1040, 1040)
    res = X.xconv_fast(H, X.XformField.rotation(T), F, X.XConvPlan(components=comps))
    assert res.standard_ops == len(comps)
    ref = orc.xconv_fast(H.astype(np.float64), ROT, T.astype(np.float64), ofilter(orc, F),
                         components=comps, nthreads=NT)[0]
    assert orc.rel_l2(res.output, ref) < TOL


@pytest.mark.parametrize("h,w,periodic", [(40, 52, False), (256, 256, False), (250, 540, False),
                                          (512, 576, True), (2030, 300, False)])
def test_cpair_fast_kernel_sizes(orc, h, w, periodic):
    """Pads without a pair plan (64, 288, 576, 512 periodic, 2048 x 324...): S2 takes
    the fast kernels' paired variant (k_fast.cu) and S4 the generic kernel's
    second, conjugated pass; band_mode reports the paired path."""
    import ctypes as C
    from paper_2006_13188_b200 import _native as N
    r, F, H, T = _rot_case(106, h, w, m_max=5, R=10)
    res = X.xconv_fast(H, X.XformField.rotation(T), F, X.XConvPlan(periodic=periodic))
    ref = orc.xconv_fast(H.astype(np.float64), ROT, T.astype(np.float64), ofilter(orc, F),
                         periodic=periodic, nthreads=NT)[0]
    assert orc.rel_l2(res.output, ref) < TOL
    # the stats of the same call through the C ABI
    ctx = N.context(0)
    out = np.zeros(H.shape, np.complex64)
    d = N.ImageDesc(h, w, 1, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_HOST, 1, 0)
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), 1, C.byref(d), H.ctypes.data,
                           T.ctypes.data, None, 0, N.XC_FLAG_PERIODIC if periodic else 0,
                           out.ctypes.data, C.byref(st)), ctx.handle)
    assert st.standard_ops == 11 and st.band_mode in (0, 2)
    if st.band_mode == 2:
        assert st.bands_run == 6
    assert np.array_equal(out, res.output)


def test_cpair_split_s2_long_columns(orc):
    """Columns of 3456 and more: G_k does not fit beside F^_k in the fast S2's
    shared memory, so S2 runs twice over the k >= 0 planes (api.cu s2_split);
    sampled pixels against the spectral oracle."""
    import ctypes as C
    from paper_2006_13188_b200 import _native as N
    r, F, _, _ = _rot_case(107, 8, 8, m_max=4, R=9)
    h, w = 3440, 500
    H = r.uniform(0, 1, (h, w)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
    ctx = N.context(0)
    out = np.zeros(H.shape, np.complex64)
    d = N.ImageDesc(h, w, 1, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_HOST, 1, 0)
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), 1, C.byref(d), H.ctypes.data,
                           T.ctypes.data, None, 0, 0, out.ctypes.data, C.byref(st)), ctx.handle)
    assert st.pad_h == 3456 and st.band_mode == 2 and st.bands_run == 5
    ys = np.concatenate([r.integers(0, h, 30), [0, h - 1]])
    xs = np.concatenate([r.integers(0, w, 30), [0, w - 1]])
    ref = orc.spectral_oracle_at(1, H, ROT, T, ofilter(orc, F), ys, xs)
    assert orc.rel_l2(out[ys, xs], ref) < TOL


def test_cpair_periodic_and_f64_signal(orc):
    r, F, H, T = _rot_case(103, 1100, 1100)
    H64, T64 = H.astype(np.float64), T.astype(np.float64)
    res = X.xconv_fast(H64, X.XformField.rotation(T64), F, X.XConvPlan(periodic=True))
    ref = orc.xconv_fast(H64, ROT, T64, ofilter(orc, F), periodic=True, nthreads=NT)[0]
    assert orc.rel_l2(res.output, ref) < TOL


def test_cpair_complex_signal_takes_full_path(orc):
    """A complex signal has no conjugate symmetry between the +k and -k
    premultiplied images; a real signal passed as complex must give the same
    output as the real one (paired path) to fp32 rounding."""
    r, F, H, T = _rot_case(104, 1030, 1030)
    Hc = H.astype(np.complex64)
    Hc.imag = r.uniform(-1, 1, H.shape).astype(np.float32)
    res = X.xconv_fast(Hc, X.XformField.rotation(T), F)
    ref = orc.xconv_fast(Hc.astype(np.complex128), ROT, T.astype(np.float64), ofilter(orc, F),
                         nthreads=NT)[0]
    assert orc.rel_l2(res.output, ref) < TOL
    a = X.xconv_fast(H, X.XformField.rotation(T), F).output
    b = X.xconv_fast(H.astype(np.complex64), X.XformField.rotation(T), F).output
    assert orc.rel_l2(a, b) < 3e-6


def test_cpair_scale_group(orc):
    """Scale group: the log-radial bands come in +-k pairs with the steering
    phase k omega log s, so the paired path applies; the inner-DC term
    (engine.hpp:369-371) is added by S4."""
    rng = orc.Rng(91)
    R = 12
    n = 1060
    OF = orc.decompose_scale2(rng.annular_filter(R), R, R, 6, 48, 32, 1.0, R)
    F = X.FreqFilter2(OF.group, OF.K, OF.ks, OF.comps, OF.n_radii, OF.n_angles, OF.r_max,
                      OF.r_min, OF.r_domain)
    r = np.random.default_rng(5)
    H = r.uniform(0, 1, (n, n)).astype(np.float32)
    S = np.exp(r.uniform(0.0, np.log(1.6), (n, n))).astype(np.float32)
    res = X.xconv_fast(H, X.XformField.scaling(S), F)
    ref = orc.xconv_fast(H.astype(np.float64), SCALE, S.astype(np.float64), OF, nthreads=NT)[0]
    assert orc.rel_l2(res.output, ref) < TOL


def test_cpair_batch_through_host_pipeline(orc):
    """A batch of real images through xc_run's host pipeline: every image on the
    paired path, each against the oracle at sampled pixels."""
    r, F, H0, T0 = _rot_case(105, 1024, 1024, m_max=4, R=10)
    B = 3
    H = r.uniform(0, 1, (B, 1024, 1024)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (B, 1024, 1024)).astype(np.float32)
    out = X.xconv_fast(H, X.XformField.rotation(T), F).output
    assert out.shape == H.shape
    ys, xs = r.integers(0, 1024, 64), r.integers(0, 1024, 64)
    for i in range(B):
        ref = orc.spectral_oracle_at(1, H[i], ROT, T[i], ofilter(orc, F), ys, xs)
        assert orc.rel_l2(out[i][ys, xs], ref) < TOL
