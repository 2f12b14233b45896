"""Packed smoothing (api.cu smooth_packable, SigMode SIG_PACK): num and den of
smooth_adaptive (engine.hpp:385-419) from ONE scatter of h w + i alpha w, with
alpha the power of two nearest max|h|.  Against the oracle at relative L2
<= 1e-5 and equal clamped-pixel counts: signal amplitudes from 1e-6 to 1e6
(alpha keeps num and den at one scale), weighted and unweighted, the scale and
rotation groups, zero signals, and a complex filter that must take the
two-scatter path.  XCB_PACK=0 reruns the two-scatter path in another process
(tests/test_gpu_fullsize.py covers config 4 at full size with packing on).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2006_13188_b200 as X

pytestmark = pytest.mark.gpu
TOL = 1e-5
SCALE, ROT = 1, 0


def ofilter(orc, F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def _scale_case(orc, n=40, R=6, seed=91):
    rng = orc.Rng(seed)
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    g = np.exp(-(x * x + y * y) / (2 * 1.8 ** 2))
    g[x * x + y * y > R * R] = 0
    F = X.decompose_scale2(g, R, R, 12, 48, 16, 0.5, R, R + 3.0)
    H = orc.gaussian_blur(rng.random_field(n, n, False).real, 2.0)
    S = rng.random_scale_field(n, n)
    return F, H, S


@pytest.mark.parametrize("amp", [1e-6, 1e-3, 1.0, 1e3, 1e6])
@pytest.mark.parametrize("normalize", [True, False])
def test_packed_scale_smoothing_any_amplitude(orc, amp, normalize):
    F, H, S = _scale_case(orc)
    Hs = H * amp
    ref, ops, cl = orc.smooth_adaptive(Hs, SCALE, S, ofilter(orc, F), normalize)
    got = X.smooth_adaptive(Hs, X.XformField.scaling(S), F, normalize_signal=normalize)
    assert orc.rel_l2(got.output, ref) < TOL, orc.rel_l2(got.output, ref)
    assert got.clamped_pixels == cl
    assert got.standard_ops == ops == 2 * F.n_components()


def test_packed_rotation_smoothing_real_filter(orc):
    """A real (Hermitian-band) rotation filter packs as well."""
    rng = orc.Rng(93)
    n, R = 36, 5
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    f = np.exp(-((x - 1.0) ** 2 + 2.0 * y * y) / 6.0)
    F = X.decompose_rotation2(f, R, R, 8, 2 * R, 32, R)
    H = rng.random_field(n, n, False).real
    T = rng.random_rotation_field(n, n)
    ref, _, cl = orc.smooth_adaptive(H, ROT, T, ofilter(orc, F))
    got = X.smooth_adaptive(H, X.XformField.rotation(T), F)
    assert orc.rel_l2(got.output, ref) < TOL and got.clamped_pixels == cl


def test_complex_filter_takes_two_scatters(orc):
    """Complex angular coefficients (F_{-k} != conj(F_k)): num and den are
    complex, so the two-scatter path runs; still the reference's answer."""
    rng = orc.Rng(94)
    n, R = 32, 5
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    f = np.exp(-(x * x + y * y) / 6.0) * (1.0 + 0.5j * np.cos(np.arctan2(y, x)))
    F = X.decompose_rotation2(f, R, R, 6, 2 * R, 32, R)
    H = rng.random_field(n, n, False).real
    T = rng.random_rotation_field(n, n)
    ref, _, cl = orc.smooth_adaptive(H, ROT, T, ofilter(orc, F))
    got = X.smooth_adaptive(H, X.XformField.rotation(T), F)
    assert orc.rel_l2(got.output, ref) < TOL and got.clamped_pixels == cl


def test_zero_signal_and_batch(orc):
    F, H, S = _scale_case(orc, n=24)
    z = X.smooth_adaptive(np.zeros_like(H), X.XformField.scaling(S), F)
    assert np.all(z.output == 0.0)
    B = np.stack([H, 3e-4 * H, np.zeros_like(H)])
    got = X.smooth_adaptive(B.astype(np.float32), X.XformField.scaling(np.stack([S] * 3)), F)
    for i in range(3):
        ref = orc.smooth_adaptive(B[i], SCALE, S, ofilter(orc, F))[0]
        if i < 2:
            assert orc.rel_l2(got.output[i], ref) < TOL
        else:
            assert np.all(got.output[i] == 0.0)


def test_pack_off_matches(orc):
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_2006_13188_b200 as X\n"
        "from paper_2006_13188_b200 import workloads as WL\n"
        "w = WL.config4(n=160)\n"
        "r = X.smooth_adaptive(w.signal[0], X.XformField.scaling(w.param[0]), w.filt)\n"
        "np.save(sys.argv[1], r.output)\n") % os.path.dirname(os.path.dirname(__file__))
    outs = []
    for flag in ("1", "0"):
        p = f"/tmp/xcb_pack_{flag}.npy"
        env = dict(os.environ, XCB_PACK=flag)
        subprocess.run([sys.executable, "-c", code, p], env=env, check=True, timeout=600)
        outs.append(np.load(p))
    assert orc.rel_l2(outs[0], outs[1]) < TOL
