"""Pins the 3D oracle restatement (oracle/xconv_oracle3d.inc) with the
reference's own known-answer tests: test_sph.cpp, test_wigner.cpp and
test_engine3d.cpp, same seeds (std::mt19937_64 fixtures of helpers.hpp), same
tolerances.  CPU only."""
import numpy as np
import pytest

PI = np.pi


def _analytic_volume(n, c, fn):  # test_sph.cpp:11-23
    z, y, x = np.mgrid[0:n, 0:n, 0:n].astype(float)
    dx, dy, dz = x - c, y - c, z - c
    r = np.sqrt(dx * dx + dy * dy + dz * dz)
    th = np.where(r > 0, np.arccos(np.clip(np.divide(dz, r, out=np.zeros_like(r), where=r > 0),
                                           -1, 1)), 0.0)
    return fn(r, th, np.arctan2(dy, dx)).astype(np.complex128)


# ---------------------------------------------------------------- test_sph.cpp

def test_sph_harm_closed_forms(orc):  # test_sph.cpp:27-42
    for th in (0.3, 1.1, 2.4):
        for ph in (0.0, 0.7, -2.0):
            assert abs(orc.sph_harm(0, 0, th, ph) - np.sqrt(1 / (4 * PI))) < 1e-13
            assert abs(orc.sph_harm(1, 0, th, ph) - np.sqrt(3 / (4 * PI)) * np.cos(th)) < 1e-13
            y11 = -np.sqrt(3 / (8 * PI)) * np.sin(th) * np.exp(1j * ph)
            assert abs(orc.sph_harm(1, 1, th, ph) - y11) < 1e-13
            assert abs(orc.sph_harm(1, -1, th, ph) + np.conj(y11)) < 1e-13
            y20 = np.sqrt(5 / (16 * PI)) * (3 * np.cos(th) ** 2 - 1)
            assert abs(orc.sph_harm(2, 0, th, ph) - y20) < 1e-13


def test_quadrature_grid_orthonormal(orc):  # test_sph.cpp:44-59
    th, w = orc.sphere_grid(8, 8)
    phis = 2 * PI * np.arange(8) / 8
    dphi = 2 * PI / 8
    Y = {(l, m): np.array([[orc.sph_harm(l, m, t, p) for p in phis] for t in th])
         for l in range(4) for m in range(-l, l + 1)}
    for a, ya in Y.items():
        for b, yb in Y.items():
            acc = np.sum(w[:, None] * dphi * ya * np.conj(yb))
            assert abs(acc - (1.0 if a == b else 0.0)) < 1e-10


def test_real_volume_hermitian_shell_coefficients(orc):  # test_sph.cpp:74-87
    rng = orc.Rng(32)
    v = np.real(rng.random_field3(11, 11, 11, False))
    f = orc.decompose_rotation3(v, 5.0, 5.0, 5.0, 3, 4, 5.0)
    for l in range(4):
        for m in range(1, l + 1):
            for j in range(f.n_radii):
                b = np.conj(f.coeff(j, l, m)) * (-1 if m % 2 else 1)
                assert abs(f.coeff(j, l, -m) - b) < 1e-10


def test_g_r_Y10_concentrates_in_one_coefficient(orc):  # test_sph.cpp:89-110
    n, c = 33, 16.0

    def g(r):
        return np.exp(-(r - 7) ** 2 / 8.0)
    v = _analytic_volume(n, c, lambda r, th, ph: g(r) * np.sqrt(3 / (4 * PI)) * np.cos(th))
    f = orc.decompose_rotation3(v, c, c, c, 2, 8, 14.0)
    assert max(abs(f.coeff(j, 1, 0)) for j in range(f.n_radii)) > 0.85
    for j in range(f.n_radii):
        r = (j + 0.5) * f.r_max / f.n_radii
        if r < 4:
            continue
        assert abs(f.coeff(j, 1, 0) - g(r)) < 5e-2
        for l in range(3):
            for m in range(-l, l + 1):
                if (l, m) != (1, 0):
                    assert abs(f.coeff(j, l, m)) < 5e-2


def test_constant_ball_is_pure_l0(orc):  # test_sph.cpp:112-124
    n, c = 25, 12.0
    v = _analytic_volume(n, c, lambda r, th, ph: np.where(r <= 11, 3.0, 0.0))
    f = orc.decompose_rotation3(v, c, c, c, 2, 6, 9.0)
    for j in range(f.n_radii):
        assert abs(f.coeff(j, 0, 0) - 3.0 * np.sqrt(4 * PI)) < 1e-6
        for l in (1, 2):
            for m in range(-l, l + 1):
                assert abs(f.coeff(j, l, m)) < 1e-8


def test_reconstruction_approximates_volume(orc):  # test_sph.cpp:126-146
    n, c = 25, 12.0

    def fn(r, th, ph):
        return np.exp(-(r - 5) ** 2 / 6.0) * (1.0 + np.cos(th) + 0.4 * np.sin(th) * np.cos(ph))
    v = _analytic_volume(n, c, fn)
    f = orc.decompose_rotation3(v, c, c, c, 2, 10, 11.0)
    back = orc.reconstruct3(f, n, n, n, c, c, c)
    z, y, x = np.mgrid[0:n, 0:n, 0:n]
    r = np.sqrt((x - c) ** 2 + (y - c) ** 2 + (z - c) ** 2)
    sel = (r >= 2) & (r <= 10)
    err = np.sqrt(np.sum(np.abs(back - v)[sel] ** 2) / np.sum(np.abs(v)[sel] ** 2))
    assert err < 8e-2


def test_angular_sampling_must_cover_band_limit(orc):  # test_sph.cpp:148-155
    v = np.zeros((9, 9, 9))
    with pytest.raises(ValueError, match="insufficient angular sampling"):
        orc.decompose_rotation3(v, 4.0, 4.0, 4.0, 3, 4, 4.0, 6, 8)
    with pytest.raises(ValueError, match="insufficient angular sampling"):
        orc.decompose_rotation3(v, 4.0, 4.0, 4.0, 3, 4, 4.0, 8, 6)


# ---------------------------------------------------------------- test_wigner.cpp

def test_wigner_identity_and_degree_zero(orc):  # test_wigner.cpp:22-37
    for l in range(5):
        assert np.abs(orc.wigner_d(l, [1, 0, 0, 0]) - np.eye(2 * l + 1)).max() < 1e-12
    rng = orc.Rng(41)
    for _ in range(5):
        assert abs(orc.wigner_d(0, rng.random_quaternion())[0, 0] - 1) < 1e-12


def _rotated_eval(q, theta, phi, fn, orc):  # test_wigner.cpp:9-18 (f(R^-1 x))
    x = np.array([np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi), np.cos(theta)])
    u = orc.quat_matrix(q).T @ x
    return fn(np.arccos(np.clip(u[2], -1, 1)), np.arctan2(u[1], u[0]))


def test_wigner_block_matches_quadrature_projection(orc):  # test_wigner.cpp:39-62
    rng = orc.Rng(42)
    l = 2
    th, w = orc.sphere_grid(8, 8)
    phis = 2 * PI * np.arange(8) / 8
    for _ in range(3):
        q = rng.random_quaternion()
        D = orc.wigner_d(l, q)
        for m in range(-l, l + 1):
            ry = np.array([[_rotated_eval(q, t, p, lambda a, b: orc.sph_harm(l, m, a, b), orc)
                            for p in phis] for t in th])
            for mp in range(-l, l + 1):
                y = np.array([[orc.sph_harm(l, mp, t, p) for p in phis] for t in th])
                acc = np.sum(w[:, None] * (2 * PI / 8) * np.conj(y) * ry)
                assert abs(acc - D[mp + l, m + l]) < 1e-8


def test_wigner_unitary_and_composition(orc):  # test_wigner.cpp:64-85
    rng = orc.Rng(43)
    for l in range(1, 5):
        for _ in range(3):
            D = orc.wigner_d(l, rng.random_quaternion())
            assert np.abs(D @ D.conj().T - np.eye(2 * l + 1)).max() < 1e-10
    rng = orc.Rng(44)
    for l in range(1, 5):
        for _ in range(3):
            a, b = rng.random_quaternion(), rng.random_quaternion()
            ab = orc.quat_mul(a, b)
            assert np.abs(orc.wigner_d(l, ab) - orc.wigner_d(l, a) @ orc.wigner_d(l, b)).max() < 1e-10


def test_wigner_z_rotations_and_degenerate_euler(orc):  # test_wigner.cpp:111-123
    for a in (0.4, -1.3, 3.0):
        q = [np.cos(a / 2), 0, 0, np.sin(a / 2)]
        D = orc.wigner_d(2, q)
        for m in range(-2, 3):
            for mp in range(-2, 3):
                want = np.exp(-1j * m * a) if m == mp else 0
                assert abs(D[m + 2, mp + 2] - want) < 1e-12


def test_wigner_validation(orc):  # test_wigner.cpp:137-142
    with pytest.raises(ValueError):
        orc.wigner_d(-1, [1, 0, 0, 0])
    with pytest.raises(ValueError, match="unit norm"):
        orc.wigner_d(1, [2.0, 0, 0, 0])


# ---------------------------------------------------------------- test_engine3d.cpp

def _decomp3(orc, vol, R, K):  # test_engine3d.cpp:9-15
    ns = max(12, 2 * (K + 1))
    return orc.decompose_rotation3(vol, R, R, R, K, 2 * R, float(R), ns, ns)


def test_identity_field_reduces_to_standard_filtering(orc):  # test_engine3d.cpp:71-87
    rng = orc.Rng(81)
    n, R = 10, 3
    F = _decomp3(orc, rng.random_smooth_filter3(R), R, 2)
    H = rng.random_field3(n, n, n, True)
    q = np.tile([1.0, 0, 0, 0], (n, n, n, 1))
    S = 2 * R + 1
    recon = orc.reconstruct3(F, S, S, S, R, R, R)
    for mode in (0, 1):
        out, _ = orc.xfast3(mode, H, q, F)
        assert orc.rel_l2(out, orc.filter3_fft(H, recon, R, R, R, mode == 0)) < 1e-10


def test_constant_rotation_matches_rotated_filter(orc):  # test_engine3d.cpp:89-115
    rng = orc.Rng(82)
    n, R, K = 10, 3, 2
    F = _decomp3(orc, rng.random_smooth_filter3(R), R, K)
    H = rng.random_field3(n, n, n, True)
    q = rng.random_quaternion()
    Frot = orc.Filter3(F.K, F.n_radii, F.r_max, F.coeffs.copy())
    for l in range(K + 1):
        D = orc.wigner_d(l, q)
        cols = [l * (l + 1) + m for m in range(-l, l + 1)]
        Frot.coeffs[:, cols] = F.coeffs[:, cols] @ D.T
    S = 2 * R + 1
    recon = orc.reconstruct3(Frot, S, S, S, R, R, R)
    qs = np.tile(q, (n, n, n, 1))
    for mode in (0, 1):
        out, _ = orc.xfast3(mode, H, qs, F)
        assert orc.rel_l2(out, orc.filter3_fft(H, recon, R, R, R, mode == 0)) < 1e-10


def test_fast_3d_matches_exact_rotated_reconstruction(orc):  # test_engine3d.cpp:139-152
    rng = orc.Rng(84)
    n, R = 8, 2
    F = _decomp3(orc, rng.random_smooth_filter3(R), R, 2)
    H = rng.random_field3(n, n, n, False)
    q = rng.random_rotation3_field(n, n, n)
    for mode in (0, 1):
        out, _ = orc.xfast3(mode, H, q, F)
        assert orc.rel_l2(out, orc.exact3(mode, H, q, F)) < 1e-8


def test_standard_convolution_count_3d(orc):  # test_engine3d.cpp:154-168
    rng = orc.Rng(85)
    n, R = 6, 2
    vol = rng.random_smooth_filter3(R)
    H = rng.random_field3(n, n, n, True)
    q = rng.random_rotation3_field(n, n, n)
    for K in (0, 2, 4):
        F = _decomp3(orc, vol, R, K)
        want = sum((2 * l + 1) ** 2 for l in range(K + 1))
        assert orc.xfast3(0, H, q, F)[1] == want
        assert orc.xfast3(1, H, q, F)[1] == want


def test_real_signal_real_filter_real_3d_response(orc):  # test_engine3d.cpp:170-185
    rng = orc.Rng(86)
    n, R = 8, 2
    F = _decomp3(orc, rng.random_smooth_filter3(R), R, 2)
    H = rng.random_field3(n, n, n, False)
    q = rng.random_rotation3_field(n, n, n)
    for mode in (0, 1):
        out, _ = orc.xfast3(mode, H, q, F)
        assert np.abs(out.imag).max() < 1e-9 * np.abs(out).max()
