"""Pin the CPU oracle to the reference's own known-answer tests.

The reference (`xconv`, /root/reference) cannot be compiled here (Eigen >= 3.4
is absent, proj/CMakeLists.txt:10), so the oracle's fidelity is established by
re-running the reference's implementation-independent KATs against it, with the
same seeded fixtures (std::mt19937_64 + std::uniform_real_distribution, as in
proj/tests/helpers.hpp) and the same tolerances.  Each test names the
reference test it ports.
"""
import itertools

import numpy as np
import pytest

ROT, SCALE = 0, 1


# --------------------------------------------------------------- test_fft.cpp

def test_fft2_round_trip(orc):  # test_fft.cpp:40-47
    rng = orc.Rng(5)
    a = rng.random_field(12, 10, True)
    b = orc.fft2(orc.fft2(a), inverse=True)
    assert orc.rel_l2(b, a) < 1e-12


def test_fft2_matches_numpy_semantics(orc):
    # kissfft semantics: forward unscaled e^-, inverse e^+ scaled 1/n (fft.hpp:19-53)
    r = np.random.default_rng(0)
    for (h, w) in [(10, 12), (27, 40), (288, 45), (1, 7), (30, 1)]:
        a = r.standard_normal((h, w)) + 1j * r.standard_normal((h, w))
        assert orc.rel_l2(orc.fft2(a), np.fft.fft2(a)) < 1e-13
        assert orc.rel_l2(orc.fft2(a, inverse=True), np.fft.ifft2(a)) < 1e-13


def test_fft_correlation_matches_direct_loop(orc):  # test_fft.cpp:49-56
    rng = orc.Rng(6)
    H = rng.random_field(13, 9, True)
    F = rng.random_field(5, 5, True)
    fast = orc.filter2_fft(H, F, 2, 2, True)
    slow = orc.correlate_direct(H, F, 2, 2)
    assert orc.rel_l2(fast, slow) < 1e-12


def test_fft_convolution_matches_direct_loop(orc):  # test_fft.cpp:58-65
    rng = orc.Rng(8)
    H = rng.random_field(8, 11, True)
    F = rng.random_field(7, 3, True)
    fast = orc.filter2_fft(H, F, 3, 1, False)
    slow = orc.convolve_direct(H, F, 3, 1)
    assert orc.rel_l2(fast, slow) < 1e-12


def test_periodic_filtering_wraps(orc):  # test_fft.cpp:67-80
    rng = orc.Rng(9)
    H = rng.random_field(8, 8, True)
    F = rng.random_field(3, 3, True)
    out = orc.filter2_fft(H, F, 1, 1, False, True)
    Hs = np.roll(H, (3, 2), axis=(0, 1))
    outs = orc.filter2_fft(Hs, F, 1, 1, False, True)
    assert np.max(np.abs(np.roll(out, (3, 2), axis=(0, 1)) - outs)) < 1e-12


def test_next_fast_size(orc):  # fft.hpp:9-17
    assert [orc.next_fast_size(n) for n in (0, 1, 7, 11, 287, 1057, 2113, 4159, 4161)] == \
        [1, 1, 8, 12, 288, 1080, 2160, 4320, 4320]


# ----------------------------------------------------------- test_engine2d.cpp

def full_decomp(orc, filt, R, n_radii=24, n_angles=64):  # test_engine2d.cpp:68-73
    return orc.decompose_rotation2(filt, R, R, n_angles, n_radii, n_angles, R)


def test_rotation_fast_matches_brute(orc):  # test_engine2d.cpp:123-138
    rng = orc.Rng(54)
    n, R = 24, 6
    F = full_decomp(orc, rng.random_smooth_filter(R), R)
    for _ in range(3):
        H = rng.random_field(n, n, False)
        T = rng.random_rotation_field(n, n)
        fc = orc.xcorr_fast(H, ROT, T, F)[0]
        assert orc.rel_l2(fc, orc.xcorr_brute(H, ROT, T, F)) < 3e-3
        fv = orc.xconv_fast(H, ROT, T, F)[0]
        assert orc.rel_l2(fv, orc.xconv_brute(H, ROT, T, F)) < 3e-3


def test_rotation_fast_matches_spectral_oracle(orc):  # test_engine2d.cpp:140-153
    rng = orc.Rng(55)
    n, R = 24, 6
    F = full_decomp(orc, rng.random_smooth_filter(R), R)
    H = rng.random_field(n, n, False)
    T = rng.random_rotation_field(n, n)
    for mode, fn in ((0, orc.xcorr_fast), (1, orc.xconv_fast)):
        assert orc.rel_l2(fn(H, ROT, T, F)[0], orc.spectral_oracle(mode, H, ROT, T, F)) < 1e-8


def test_constant_rotation_is_rotated_filtering(orc):  # test_engine2d.cpp:155-174
    rng = orc.Rng(56)
    n, R = 20, 5
    F = full_decomp(orc, rng.random_smooth_filter(R), R, 20, 64)
    th0 = 0.9
    Frot = orc.Filter(**{**F.__dict__, "comps": F.comps * np.exp(-1j * np.asarray(F.ks) * th0)})
    rot = orc.reconstruct(Frot, 2 * R + 1, 2 * R + 1, R, R)
    H = rng.random_field(n, n, True)
    T = np.full((n, n), th0)
    assert orc.rel_l2(orc.xcorr_fast(H, ROT, T, F)[0], orc.filter2_fft(H, rot, R, R, True)) < 1e-10
    assert orc.rel_l2(orc.xconv_fast(H, ROT, T, F)[0], orc.filter2_fft(H, rot, R, R, False)) < 1e-10


def test_single_component_plan(orc):  # test_engine2d.cpp:176-194
    rng = orc.Rng(57)
    n, R = 16, 5
    F = full_decomp(orc, rng.random_smooth_filter(R), R, 16, 32)
    H = rng.random_field(n, n, True)
    T = rng.random_rotation_field(n, n)
    out, ops, _ = orc.xcorr_fast(H, ROT, T, F, components=[2])
    assert ops == 1
    F2 = orc.render_component(F, F.index_of(2), 2 * R + 1, 2 * R + 1, R, R)
    G = orc.filter2_fft(H, F2, R, R, True)
    assert orc.rel_l2(out, G * np.exp(2j * T)) < 1e-12


def test_periodic_translation_equivariance(orc):  # test_engine2d.cpp:196-219
    rng = orc.Rng(58)
    n, R = 16, 4
    F = full_decomp(orc, rng.random_smooth_filter(R), R, 12, 32)
    H = rng.random_field(n, n, True)
    T = rng.random_rotation_field(n, n)
    base = orc.xcorr_fast(H, ROT, T, F, periodic=True)[0]
    sh = orc.xcorr_fast(np.roll(H, (3, 5), (0, 1)), ROT, np.roll(T, (3, 5), (0, 1)), F,
                        periodic=True)[0]
    assert np.max(np.abs(np.roll(base, (3, 5), (0, 1)) - sh)) < 1e-10


def test_standard_op_count(orc):  # test_engine2d.cpp:221-235
    rng = orc.Rng(59)
    n, R = 12, 4
    filt = rng.random_smooth_filter(R)
    H = rng.random_field(n, n, True)
    T = rng.random_rotation_field(n, n)
    for K in (0, 2, 4, 8):
        F = orc.decompose_rotation2(filt, R, R, K, 12, 32, R)
        assert orc.xcorr_fast(H, ROT, T, F)[1] == 2 * (K // 2) + 1
        assert orc.xconv_fast(H, ROT, T, F)[1] == 2 * (K // 2) + 1


def test_real_in_real_out(orc):  # test_engine2d.cpp:237-248
    rng = orc.Rng(60)
    n, R = 18, 5
    F = full_decomp(orc, rng.random_smooth_filter(R), R, 16, 32)
    H = rng.random_field(n, n, False)
    T = rng.random_rotation_field(n, n)
    for fn in (orc.xcorr_fast, orc.xconv_fast):
        out = fn(H, ROT, T, F)[0]
        assert np.max(np.abs(out.imag)) < 1e-9 * np.max(np.abs(out))


def test_truncation_optimality(orc):  # test_engine2d.cpp:250-283
    rng = orc.Rng(61)
    R = 5
    F = orc.decompose_rotation2(rng.random_smooth_filter(R), R, R, 6, 16, 64, R)
    assert F.n_components() == 7
    full = orc.synthesize_polar(F)

    def subset_error(mask):
        keep = [int(F.ks[c]) for c in range(7) if mask & (1 << c)]
        part = orc.synthesize_polar(F, keep)
        return float(np.sum(np.abs(part - full) ** 2))

    energy = np.sum(np.abs(F.comps) ** 2, axis=0)
    order = sorted(range(7), key=lambda i: -energy[i])
    for m in range(1, 7):
        best = subset_error(sum(1 << order[i] for i in range(m)))
        for combo in itertools.combinations(range(7), m):
            assert best <= subset_error(sum(1 << c for c in combo)) + 1e-12


def test_input_validation(orc):  # test_engine2d.cpp:285-299
    rng = orc.Rng(62)
    R = 4
    F = full_decomp(orc, rng.random_smooth_filter(R), R, 8, 16)
    H = rng.random_field(10, 10, True)
    with pytest.raises(ValueError, match="group mismatch"):
        orc.xcorr_fast(H, SCALE, np.ones((10, 10)), F)
    T = rng.random_rotation_field(10, 10)
    with pytest.raises(ValueError, match="plan retains a component the filter lacks"):
        orc.xcorr_fast(H, ROT, T, F, components=[99])


# ------------------------------------------------------- test_engine_scale.cpp

def scale_decomp(orc, filt, R, K, r_min, n_radii=48, n_angles=32):  # :30-34
    return orc.decompose_scale2(filt, R, R, K, n_radii, n_angles, r_min, R)


def test_unit_scale_is_standard_filtering(orc):  # test_engine_scale.cpp:82-96
    rng = orc.Rng(71)
    n, R = 20, 6
    F = scale_decomp(orc, rng.annular_filter(R), R, 48, 1.0)
    recon = orc.reconstruct(F, 2 * R + 1, 2 * R + 1, R, R)
    H = rng.random_field(n, n, True)
    T = np.ones((n, n))
    assert orc.rel_l2(orc.xcorr_fast(H, SCALE, T, F)[0], orc.filter2_fft(H, recon, R, R, True)) < 1e-10
    assert orc.rel_l2(orc.xconv_fast(H, SCALE, T, F)[0], orc.filter2_fft(H, recon, R, R, False)) < 1e-10


@pytest.mark.slow
def test_scale_fast_matches_brute(orc):  # test_engine_scale.cpp:98-119
    rng = orc.Rng(72)
    n, R = 24, 8
    F = scale_decomp(orc, rng.annular_filter(R, 0.354, 0.044), R, 46, 1.0)
    for _ in range(3):
        H = rng.random_field(n, n, False)
        T = rng.random_scale_field(n, n)
        assert orc.rel_l2(orc.xcorr_fast(H, SCALE, T, F)[0], orc.xcorr_brute(H, SCALE, T, F)) < 3e-3
        assert orc.rel_l2(orc.xconv_fast(H, SCALE, T, F)[0], orc.xconv_brute(H, SCALE, T, F)) < 3e-3


def test_scale_fast_matches_spectral_oracle(orc):  # test_engine_scale.cpp:121-134
    rng = orc.Rng(73)
    n, R = 20, 6
    F = scale_decomp(orc, rng.annular_filter(R), R, 8, 1.0)
    H = rng.random_field(n, n, False)
    T = rng.random_scale_field(n, n)
    for mode, fn in ((0, orc.xcorr_fast), (1, orc.xconv_fast)):
        assert orc.rel_l2(fn(H, SCALE, T, F)[0], orc.spectral_oracle(mode, H, SCALE, T, F)) < 1e-8


def test_scale_op_count(orc):  # test_engine_scale.cpp:136-147
    rng = orc.Rng(74)
    n, R = 12, 5
    filt = rng.annular_filter(R)
    H = rng.random_field(n, n, True)
    T = rng.random_scale_field(n, n)
    for K in (0, 2, 4, 8):
        F = scale_decomp(orc, filt, R, K, 1.0)
        assert orc.xcorr_fast(H, SCALE, T, F)[1] == 2 * (K // 2) + 1
        assert orc.xconv_fast(H, SCALE, T, F)[1] == 2 * (K // 2) + 1


def test_scale_real_in_real_out(orc):  # test_engine_scale.cpp:149-159
    rng = orc.Rng(75)
    n, R = 16, 5
    F = scale_decomp(orc, rng.annular_filter(R), R, 8, 1.0)
    H = rng.random_field(n, n, False)
    T = rng.random_scale_field(n, n)
    for fn in (orc.xcorr_fast, orc.xconv_fast):
        out = fn(H, SCALE, T, F)[0]
        assert np.max(np.abs(out.imag)) < 1e-9 * np.max(np.abs(out))


def test_scale_guard_band_names_pixel(orc):  # test_engine_scale.cpp:161-178
    rng = orc.Rng(76)
    n, R = 8, 5
    F = scale_decomp(orc, rng.annular_filter(R), R, 4, 1.0)
    H = rng.random_field(n, n, True)
    s = np.ones((n, n))
    s[3, 5] = 10.0
    with pytest.raises(ValueError) as ei:
        orc.xcorr_fast(H, SCALE, s, F)
    assert "guard band" in str(ei.value) and "(5,3)" in str(ei.value)


# ------------------------------------------------------------ test_smooth.cpp

def gaussian_filter(R, sigma):  # test_smooth.cpp:9-18
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    f = np.exp(-(x * x + y * y) / (2 * sigma * sigma))
    f[x * x + y * y > R * R] = 0
    return f.astype(np.complex128)


def gaussian_scale_filter(orc, R, sigma):  # test_smooth.cpp:20-27
    return orc.decompose_scale2(gaussian_filter(R, sigma), R, R, 62, 64, 16, 0.5, R, R + 3.0)


def smooth_image(orc, rng, n, sigma=2.0):  # test_smooth.cpp:29-38
    return orc.gaussian_blur(rng.random_field(n, n, False).real, sigma).astype(np.complex128)


def steered_kernel(orc, F, s):  # test_smooth.cpp:40-65
    R = int(np.ceil(F.r_max))
    w = F.omega()
    k = np.zeros((2 * R + 1, 2 * R + 1), np.complex128)
    dc = orc.inner_dc_value(F)
    for y in range(-R, R + 1):
        for x in range(-R, R + 1):
            r = np.hypot(x, y)
            if r > F.r_max:
                continue
            if r < F.r_min:
                k[y + R, x + R] = dc
                continue
            th = np.arctan2(y, x)
            k[y + R, x + R] = sum(orc.component_value(F, ci, r, th) *
                                  np.exp(-1j * F.ks[ci] * w * np.log(s))
                                  for ci in range(F.n_components()))
    return k


def tile_blur(orc, H, R, k):  # test_smooth.cpp:67-74
    num = orc.filter2_fft(H, k, R, R, False)
    den = orc.filter2_fft(np.ones_like(H), k, R, R, False)
    return (num / den).real


def checker_field(n, tile, s0, s1):  # test_smooth.cpp:76-83
    y, x = np.mgrid[0:n, 0:n]
    return np.where(((x // tile + y // tile) % 2) == 0, s0, s1).astype(np.float64)


def interior_rel(a, T, tile, margin, truths, scales):  # test_smooth.cpp:85-104
    n = a.shape[0]
    y, x = np.mgrid[0:n, 0:n]
    bx, by = x % tile, y % tile
    m = (bx >= margin) & (by >= margin) & (bx < tile - margin) & (by < tile - margin)
    t = np.where(T == scales[0], truths[0], truths[1])
    return float(np.sqrt(np.sum(((a - t) ** 2)[m]) / np.sum((t ** 2)[m])))


def test_smooth_constant_fixed_point(orc):  # test_smooth.cpp:108-123
    rng = orc.Rng(91)
    n, R = 32, 6
    F = gaussian_scale_filter(orc, R, 1.8)
    H = np.full((n, n), 0.7, np.complex128)
    out = orc.smooth_adaptive(H, SCALE, rng.random_scale_field(n, n), F)[0]
    assert np.max(np.abs(out - 0.7)) < 1e-6
    aniso = np.abs(rng.random_smooth_filter(R)) + 0.05
    Fr = orc.decompose_rotation2(aniso, R, R, 8, 2 * R, 32, R)
    outr = orc.smooth_adaptive(H, ROT, rng.random_rotation_field(n, n), Fr)[0]
    assert np.max(np.abs(outr - 0.7)) < 1e-6


def test_smooth_unit_scale_is_normalized_blur(orc):  # test_smooth.cpp:125-137
    rng = orc.Rng(92)
    n, R = 32, 6
    F = gaussian_scale_filter(orc, R, 1.8)
    H = smooth_image(orc, rng, n)
    out = orc.smooth_adaptive(H, SCALE, np.ones((n, n)), F)[0]
    recon = orc.reconstruct(F, 2 * R + 1, 2 * R + 1, R, R)
    num = orc.filter2_fft(H, recon, R, R, False)
    den = orc.filter2_fft(np.ones_like(H), recon, R, R, False)
    assert orc.rel_l2(out, num / den) < 1e-6


@pytest.mark.slow
def test_smooth_checkerboard_and_bleeding(orc):  # test_smooth.cpp:139-172
    for seed, check_bleed in ((93, False), (94, True)):
        rng = orc.Rng(seed)
        n, tile, R = 64, 32, 8
        sigma, s0, s1 = 2.0, 0.8, 1.3
        F = gaussian_scale_filter(orc, R, sigma)
        H = smooth_image(orc, rng, n)
        T = checker_field(n, tile, s0, s1)
        truths = [tile_blur(orc, H, R, steered_kernel(orc, F, s)) for s in (s0, s1)]
        good = orc.smooth_adaptive(H, SCALE, T, F, True)[0]
        if not check_bleed:
            assert interior_rel(good, T, tile, R, truths, (s0, s1)) < 3e-3
        else:
            bad = orc.smooth_adaptive(H, SCALE, T, F, False)[0]
            assert interior_rel(bad, T, tile, 0, truths, (s0, s1)) > \
                interior_rel(good, T, tile, 0, truths, (s0, s1))


def test_smooth_zero_integral_rejected(orc):  # test_smooth.cpp:174-187
    rng = orc.Rng(95)
    n, R = 16, 5
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    f = (x * np.exp(-(x * x + y * y) / 8.0)).astype(np.complex128)
    F = orc.decompose_rotation2(f, R, R, 8, 2 * R, 32, R)
    H = rng.random_field(n, n, False)
    with pytest.raises(ValueError, match="normalization undefined"):
        orc.smooth_adaptive(H, ROT, rng.random_rotation_field(n, n), F)


# ------------------------------------------------------------ acceptance.cpp

def steered_recon(orc, F, param):  # acceptance.cpp:81-105
    R = int(np.ceil(F.r_max))
    k = np.zeros((2 * R + 1, 2 * R + 1), np.complex128)
    w = F.omega() if F.group == SCALE else 0.0
    dc = orc.inner_dc_value(F) if F.group == SCALE else 0
    for y in range(-R, R + 1):
        for x in range(-R, R + 1):
            r = np.hypot(x, y)
            if r > F.r_max:
                continue
            if F.group == SCALE and r < F.r_min:
                k[y + R, x + R] = dc
                continue
            th = np.arctan2(y, x)
            acc = 0
            for ci in range(F.n_components()):
                ph = -F.ks[ci] * param if F.group == ROT else -F.ks[ci] * w * np.log(param)
                acc += orc.component_value(F, ci, r, th) * np.exp(1j * ph)
            k[y + R, x + R] = acc
    return k


def test_acceptance_criterion5_constant_fields(orc):  # acceptance.cpp:297-335
    rng = orc.Rng(205)
    n, R = 20, 6
    worst_t = worst_id = 0.0
    F = orc.decompose_rotation2(rng.random_smooth_filter(R), R, R, 64, 24, 64, R)
    H = rng.random_field(n, n, True)
    rot = steered_recon(orc, F, 0.9)
    fast = orc.xcorr_fast(H, ROT, np.full((n, n), 0.9), F)[0]
    worst_t = max(worst_t, orc.rel_l2(fast, orc.filter2_fft(H, rot, R, R, True)))
    recon = orc.reconstruct(F, 2 * R + 1, 2 * R + 1, R, R)
    idr = orc.xconv_fast(H, ROT, np.zeros((n, n)), F)[0]
    worst_id = max(worst_id, orc.rel_l2(idr, orc.filter2_fft(H, recon, R, R, False)))
    F = orc.decompose_scale2(rng.annular_filter(R, 0.354, 0.044), R, R, 34, 36, 32, 1.0, R)
    H = rng.random_field(n, n, True)
    sc = steered_recon(orc, F, 1.4)
    fast = orc.xconv_fast(H, SCALE, np.full((n, n), 1.4), F)[0]
    worst_t = max(worst_t, orc.rel_l2(fast, orc.filter2_fft(H, sc, R, R, False)))
    recon = orc.reconstruct(F, 2 * R + 1, 2 * R + 1, R, R)
    ids = orc.xcorr_fast(H, SCALE, np.ones((n, n)), F)[0]
    worst_id = max(worst_id, orc.rel_l2(ids, orc.filter2_fft(H, recon, R, R, True)))
    assert worst_t <= 1e-3 and worst_id <= 1e-6


def test_acceptance_criterion6_delta(orc):  # acceptance.cpp:337-361
    rng = orc.Rng(206)
    R = 6
    n = 2 * R + 1
    F = orc.decompose_rotation2(rng.random_smooth_filter(R), R, R, 64, 24, 64, R)
    delta = np.zeros((n, n), np.complex128)
    delta[R, R] = 1.0
    resp = orc.xconv_fast(delta, ROT, np.full((n, n), 0.7), F)[0]
    worst = orc.rel_l2(resp, steered_recon(orc, F, 0.7))
    F = orc.decompose_scale2(rng.annular_filter(R, 0.354, 0.044), R, R, 34, 36, 32, 1.0, R)
    resp = orc.xconv_fast(delta, SCALE, np.full((n, n), 1.3), F)[0]
    worst = max(worst, orc.rel_l2(resp, steered_recon(orc, F, 1.3)))
    assert worst <= 1e-3


# ------------------------------------------------------- new: angle max (A9)

def test_anglemax_matches_direct_numpy(orc):
    r = np.random.default_rng(3)
    ks = np.arange(-4, 5)
    G = r.standard_normal((9, 5, 6)) + 1j * r.standard_normal((9, 5, 6))
    score, arg = orc.anglemax(G, ks, 360)
    s = np.arange(360)
    ph = np.exp(-2j * np.pi * np.outer(s, ks) / 360)        # (360, nc)
    X = np.abs(np.einsum("sk,kyx->syx", ph, G))
    assert np.allclose(score, X.max(0), rtol=1e-12)
    assert np.array_equal(arg, X.argmax(0))


def test_find_peaks_tie_break(orc):  # vote_filter.hpp:107-134
    resp = np.zeros((9, 9))
    resp[2, 2] = resp[2, 6] = 1.0  # equal values: sorted by y then x
    resp[6, 4] = 2.0
    resp[6, 5] = 2.0               # plateau: left/up neighbour wins
    pk = orc.find_peaks(resp, 1.5, 0.4)
    assert pk == [(4, 6, 2.0), (2, 2, 1.0), (6, 2, 1.0)]
