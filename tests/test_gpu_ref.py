"""GPU parity against the REFERENCE implementation itself (oracle/_ref: the
reference's headers compiled unchanged against the Eigen-subset shim, its own
test suite green in tests/test_ref_suite.py), on the BASELINE configs'
seeded inputs: reduced image sizes for every config, full size for configs 1
and 2.  Tolerance: relative L2 <= 1e-5 (fp32 GPU vs the reference's double);
peak lists and argmax at the peaks exact.
"""
import os

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from oracle import refimpl
from paper_2006_13188_b200 import workloads as WL

pytestmark = pytest.mark.gpu
TOL = 1e-5
NT = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def ref():
    refimpl.build()  # prebuilt oracle/_ref on the GPU box
    assert refimpl.available(), "oracle/_ref missing: build it with `make -C oracle ref`"
    return refimpl


def decompose(mod, w):
    group, args = w.decomp
    fn = mod.decompose_rotation2 if group == "rotation2" else mod.decompose_scale2
    return fn(w.filter_image, *args)


def pfilter(F):
    return X.FreqFilter2(F.group, F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max, F.r_min,
                         F.r_domain)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("cfg,n", [(1, 256), (2, 1024), (5, 160), (1, 97)])
def test_gather_scatter_vs_reference(ref, cfg, n):
    w = WL.config5(n=n, batch=1) if cfg == 5 else WL.CONFIGS[cfg](n=n)
    R = decompose(ref, w)  # the reference's decomposition feeds both sides
    mode = 0 if w.mode == "xcorr" else 1
    got = (X.xcorr_fast if mode == 0 else X.xconv_fast)(
        w.signal[0], X.XformField.rotation(w.param[0]), pfilter(R))
    want, ops = ref.xfast(mode, w.signal[0].astype(np.float64), 0,
                          w.param[0].astype(np.float64), R, nthreads=NT)
    assert got.standard_ops == ops
    assert rel(got.output, want) < TOL


def test_scale_smoothing_vs_reference(ref):
    w = WL.config4(n=192)
    R = decompose(ref, w)
    H, S = w.signal[0], w.param[0]
    got = X.smooth_adaptive(H, X.XformField.scaling(S), pfilter(R))
    want, ops, cl = ref.smooth_adaptive(H.astype(np.float64), 1, S.astype(np.float64), R)
    assert got.standard_ops == ops and got.clamped_pixels == cl
    assert rel(got.output, want) < TOL
    for mode in (0, 1):
        g = (X.xcorr_fast if mode == 0 else X.xconv_fast)(H, X.XformField.scaling(S), pfilter(R))
        r, _ = ref.xfast(mode, H.astype(np.float64), 1, S.astype(np.float64), R, nthreads=NT)
        assert rel(g.output, r) < TOL


def test_anglemax_peaks_vs_reference(ref, orc):
    """Config 3 at 512^2 with two pasted templates: the GPU score and find_peaks
    list vs the reference's per-band correlations (single-band xcorr_fast, zero
    angle field) -> angle max -> the reference's find_peaks."""
    w = WL.config3(n=512, n_templates=2)
    R = decompose(ref, w)
    H = w.signal[0].astype(np.float64)
    zero = np.zeros_like(H)
    G = np.stack([ref.xcorr_fast(H, 0, zero, R, [int(k)])[0] for k in R.ks])
    oscore, oarg = orc.anglemax_mt(G, R.ks, 360, nthreads=NT)
    score, arg = X.anglemax(w.signal[0], pfilter(R), 360)
    assert rel(score, oscore) < TOL
    want = ref.find_peaks(oscore, 32.0, 0.5)
    got = X.find_peaks(score.astype(np.float64), 32.0, 0.5)
    assert [(p.x, p.y) for p in got[:2]] == [(x, y) for x, y, _ in want[:2]]
    for x, y, _ in want[:2]:
        assert arg[y, x] == oarg[y, x]


def test_detect_pattern_vs_reference(ref):
    r = np.random.default_rng(5)
    Rr = 12
    y, x = np.mgrid[-Rr:Rr + 1, -Rr:Rr + 1].astype(np.float64)
    pat = (np.exp(-((x - 4) ** 2 + (y + 3) ** 2) / 12.0) -
           0.8 * np.exp(-((x + 5) ** 2 + (y - 3) ** 2) / 9.0)) * np.exp(-(x * x + y * y) / 120.0)
    img = r.normal(0, 0.02, (256, 320))
    for cx, cy, a in ((80.0, 90.0, 0.4), (230.0, 170.0, 2.1), (150.0, 60.0, -1.0)):
        WL.paste_rotated(img, pat, cx, cy, a)
    resp, pk, ops = ref.detect_pattern(pat, Rr, Rr, float(Rr), img, 24)
    vf = X.build_optimal_filter(pat, Rr, Rr, float(Rr))
    det = X.detect_pattern(img, vf, 24)
    assert det.standard_ops == ops
    assert rel(det.response, resp) < TOL
    assert [(p.x, p.y) for p in det.peaks[:3]] == [(a, b) for a, b, _ in pk[:3]]
