"""3D rotation pipeline: the host decomposition against the
oracle (CPU), and xcorr_fast_3d / xconv_fast_3d on the GPU against the oracle
restatement of engine3d.hpp and the reference's 3D known-answer tests
(test_engine3d.cpp), relative L2 <= 1e-5 (fp32 GPU vs fp64 oracle)."""
import numpy as np
import pytest

import paper_2006_13188_b200 as X

TOL = 1e-5


def _filters(orc, vol, R, K, ns=None):
    ns = ns or max(12, 2 * (K + 1))
    F = orc.decompose_rotation3(vol, R, R, R, K, 2 * R, float(R), ns, ns)
    G = X.decompose_rotation3(vol, R, R, R, K, 2 * R, float(R), ns, ns)
    return F, G


# ---------------------------------------------------------------- host (CPU)

def test_host_decomposition_render_wigner_match_oracle(orc):
    rng = orc.Rng(91)
    R = 3
    vol = rng.random_smooth_filter3(R)
    F, G = _filters(orc, vol, R, 3)
    assert np.abs(F.coeffs - G.coeffs).max() < 1e-12 * np.abs(F.coeffs).max()
    S = 2 * R + 1
    for l, m, mp in ((0, 0, 0), (2, -1, 2), (3, 3, -2)):
        a = orc.render_sph_component(F, l, m, mp, S, S, S, R, R, R)
        b = X.render_sph_component(G, l, m, mp, S, S, S, R, R, R)
        assert np.abs(a - b).max() < 1e-12
    a = orc.reconstruct3(F, 9, 8, 7, 4.0, 3.5, 3.0, degrees=[0, 2])
    b = X.reconstruct3(G, 9, 8, 7, 4.0, 3.5, 3.0, degrees=[0, 2])
    assert np.abs(a - b).max() < 1e-12
    for _ in range(3):
        q = rng.random_quaternion()
        for l in range(6):
            assert np.abs(orc.wigner_d(l, q) - X.wigner_d(l, q)).max() < 1e-12
    for q in ([1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [np.cos(0.3), 0, 0, np.sin(0.3)]):
        for l in (1, 3):
            assert np.abs(orc.wigner_d(l, q) - X.wigner_d(l, q)).max() < 1e-12
    assert abs(orc.sph_harm(4, -3, 0.7, -1.1) - X.sph_harm(4, -3, 0.7, -1.1)) < 1e-14


def test_host_validation_texts():
    v = np.zeros((9, 9, 9))
    with pytest.raises(ValueError, match="insufficient angular sampling for band limit"):
        X.decompose_rotation3(v, 4.0, 4.0, 4.0, 3, 4, 4.0, 6, 8)
    with pytest.raises(ValueError, match="degree must be >= 0"):
        X.wigner_d(-1, [1, 0, 0, 0])
    with pytest.raises(ValueError, match="rotation quaternion must be unit norm"):
        X.wigner_d(1, [2.0, 0, 0, 0])
    with pytest.raises(ValueError, match=r"\|m\| must be <= l"):
        X.sph_harm(1, 2, 0.1, 0.2)


def test_3d_hot_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    F = X.SphFilter3(0, 2, 2.0, np.ones((2, 1)))
    with pytest.raises(RuntimeError):
        X.xcorr_fast_3d(np.zeros((4, 4, 4)), X.rotation3d(np.tile([1.0, 0, 0, 0], (4, 4, 4, 1))),
                        F)


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("complex_signal", [False, True])
def test_fast_3d_matches_oracle(orc, complex_signal):
    rng = orc.Rng(83)
    n, R = 12, 3
    F, G = _filters(orc, rng.random_smooth_filter3(R), R, 2)
    H = rng.random_field3(n, n, n, complex_signal)
    q = rng.random_rotation3_field(n, n, n)
    T = X.rotation3d(q)
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        r = fn(H if complex_signal else H.real, T, G)
        ref, ops = orc.xfast3(mode, H, q, F)
        assert r.standard_ops == ops == 35
        assert r.gpu_launches > 0
        assert orc.rel_l2(r.output, ref) < TOL, (mode, orc.rel_l2(r.output, ref))


@pytest.mark.gpu
def test_identity_and_constant_rotation_reduce_to_standard_filtering(orc):
    # test_engine3d.cpp:71-115
    rng = orc.Rng(82)
    n, R, K = 10, 3, 2
    F, G = _filters(orc, rng.random_smooth_filter3(R), R, K)
    H = rng.random_field3(n, n, n, True)
    S = 2 * R + 1
    ident = np.tile([1.0, 0, 0, 0], (n, n, n, 1))
    recon = orc.reconstruct3(F, S, S, S, R, R, R)
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        out = fn(H, X.rotation3d(ident), G).output
        assert orc.rel_l2(out, orc.filter3_fft(H, recon, R, R, R, mode == 0)) < TOL
    q = rng.random_quaternion()
    Frot = orc.Filter3(F.K, F.n_radii, F.r_max, F.coeffs.copy())
    for l in range(K + 1):
        cols = [l * (l + 1) + m for m in range(-l, l + 1)]
        Frot.coeffs[:, cols] = F.coeffs[:, cols] @ orc.wigner_d(l, q).T
    recon = orc.reconstruct3(Frot, S, S, S, R, R, R)
    T = X.rotation3d(np.tile(q, (n, n, n, 1)))
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        out = fn(H, T, G).output
        assert orc.rel_l2(out, orc.filter3_fft(H, recon, R, R, R, mode == 0)) < TOL


@pytest.mark.gpu
def test_fast_3d_matches_exact_rotated_reconstruction(orc):  # test_engine3d.cpp:139-152
    rng = orc.Rng(84)
    n, R = 8, 2
    F, G = _filters(orc, rng.random_smooth_filter3(R), R, 2)
    H = rng.random_field3(n, n, n, False)
    q = rng.random_rotation3_field(n, n, n)
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        out = fn(H.real, X.rotation3d(q), G).output
        assert orc.rel_l2(out, orc.exact3(mode, H, q, F)) < TOL
        assert np.abs(out.imag).max() < 1e-5 * np.abs(out).max()  # real in, real out


@pytest.mark.gpu
def test_3d_counts_degree_subsets_and_ragged_volumes(orc):
    rng = orc.Rng(85)
    R = 2
    vol = rng.random_smooth_filter3(R)
    nx, ny, nz = 9, 7, 12
    H = rng.random_field3(nx, ny, nz, True)
    q = rng.random_rotation3_field(nx, ny, nz)
    T = X.rotation3d(q)
    for K in (0, 2, 4):
        F, G = _filters(orc, vol, R, K)
        want = sum((2 * l + 1) ** 2 for l in range(K + 1))
        assert X.xcorr_fast_3d(H, T, G).standard_ops == want
        assert X.xconv_fast_3d(H, T, G).standard_ops == want
    F, G = _filters(orc, vol, R, 4)
    plan = X.XConvPlan(components=[1, 3])
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        r = fn(H, T, G, plan)
        ref, ops = orc.xfast3(mode, H, q, F, degrees=[1, 3])
        assert r.standard_ops == ops == 9 + 49
        assert orc.rel_l2(r.output, ref) < TOL
    with pytest.raises(ValueError, match="plan retains a component the filter lacks"):
        X.xcorr_fast_3d(H, T, G, X.XConvPlan(components=[5]))


@pytest.mark.gpu
def test_3d_tiny_volumes_and_non_unit_quaternions(orc):
    rng = orc.Rng(87)
    R = 2
    F, G = _filters(orc, rng.random_smooth_filter3(R), R, 2)
    for shape in ((1, 1, 1), (1, 3, 2), (5, 1, 4)):
        nz, ny, nx = shape
        H = rng.random_field3(nx, ny, nz, True)
        q = rng.random_rotation3_field(nx, ny, nz) * 1.7  # renormalized (field.hpp:168-171)
        for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
            out = fn(H, X.rotation3d(q), G).output
            ref, _ = orc.xfast3(mode, H, q, F)
            assert orc.rel_l2(out, ref) < TOL, (shape, mode)


@pytest.mark.gpu
def test_3d_validation():  # test_engine3d.cpp:187-197
    G = X.SphFilter3(2, 4, 2.0, np.ones((4, 9)))
    H = np.zeros((6, 6, 6))
    with pytest.raises(ValueError, match="needs a rotation3 field"):
        X.xcorr_fast_3d(H, X.XformField.rotation(np.zeros((6, 6))), G)
    with pytest.raises(ValueError, match="signal and transformation field dims differ"):
        X.xconv_fast_3d(H, X.rotation3d(np.tile([1.0, 0, 0, 0], (5, 6, 6, 1))), G)


@pytest.mark.gpu
def test_fast_3d_larger_volume_higher_band_limit(orc):
    rng = orc.Rng(88)
    n, R, K = 24, 4, 4
    F, G = _filters(orc, rng.random_smooth_filter3(R), R, K)
    H = rng.random_field3(n, n, n, False)
    q = rng.random_rotation3_field(n, n, n)
    T = X.rotation3d(q)
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        r = fn(H.real, T, G)
        ref, ops = orc.xfast3(mode, H, q, F)
        assert r.standard_ops == ops == 165
        assert orc.rel_l2(r.output, ref) < TOL, (mode, orc.rel_l2(r.output, ref))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("XCB_FUZZ_CASES", "12"))))
def test_fast_3d_random_cases(orc, seed):
    """Random 3D geometries (ragged, thin), degree limits, degree subsets, real and
    complex signals against the oracle."""
    r = np.random.default_rng([seed, 3003])
    R = int(r.integers(1, 5))
    K = int(r.integers(0, 5))
    nx, ny, nz = (int(v) for v in r.integers(1, 18, 3))
    rng = orc.Rng(1000 + seed)
    F, G = _filters(orc, rng.random_smooth_filter3(R), R, K)
    cplx = bool(r.random() < 0.5)
    H = rng.random_field3(nx, ny, nz, cplx)
    q = rng.random_rotation3_field(nx, ny, nz)
    degrees = None
    if K > 0 and r.random() < 0.4:
        degrees = sorted(r.choice(np.arange(K + 1), size=int(r.integers(1, K + 2)),
                                  replace=False).tolist())
    plan = X.XConvPlan(components=degrees or [])
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        got = fn(H if cplx else H.real, X.rotation3d(q), G, plan)
        ref, ops = orc.xfast3(mode, H, q, F, degrees=degrees)
        assert got.standard_ops == ops
        err = orc.rel_l2(got.output, ref)
        assert err < TOL, (seed, mode, (nx, ny, nz), R, K, degrees, err)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,degrees", [((68, 64, 60), [0, 1]), ((76, 86, 70), [1]),
                                          ((128, 131, 140), [0])])
def test_3d_compile_time_tile_plans(orc, dims, degrees):
    """Pads with compile-time tile plans (k_3d.cu CtPlan): 72 = 9·8, 80 = 10·8,
    90 = 10·9 (two passes), 135 = 9·5·3 and 144 = 6·6·4 (three passes), mixed
    with runtime-plan axes (64 = 8·8), against the oracle on a degree subset."""
    rng = orc.Rng(87)
    R = 4
    F, G = _filters(orc, rng.random_smooth_filter3(R), R, 2)
    nx, ny, nz = dims
    H = rng.random_field3(nx, ny, nz, False)
    q = rng.random_rotation3_field(nx, ny, nz)
    T = X.rotation3d(q)
    plan = X.XConvPlan(components=degrees)
    for mode, fn in ((0, X.xcorr_fast_3d), (1, X.xconv_fast_3d)):
        r = fn(H.real, T, G, plan)
        ref, ops = orc.xfast3(mode, H, q, F, degrees=degrees)
        assert r.standard_ops == ops == sum((2 * l + 1) ** 2 for l in degrees)
        assert orc.rel_l2(r.output, ref) < TOL, (mode, orc.rel_l2(r.output, ref))
