"""Parity pin on the CPU: the oracle's restatement (oracle/xconv_oracle.cpp) and
the product's host C++ (csrc/host_filter.cpp, through the C ABI's host entry
points) against the REFERENCE implementation itself (oracle/_ref, the
reference's headers compiled unchanged; tests/test_ref_suite.py shows its own
test suite passes).  Inputs are the BASELINE configs' seeded workloads at
reduced image sizes (the filters are the full-size ones).

Both sides compute in double with the same kissfft-ordered FFT, so the bound
is 1e-12 relative L2 (1e-13 for the host decompositions, which share no code
with the reference but follow the same arithmetic), and peak lists are equal.
"""
import numpy as np
import pytest

import paper_2006_13188_b200 as X
from oracle import refimpl
from paper_2006_13188_b200 import workloads as WL

TIGHT = 1e-12


@pytest.fixture(scope="module")
def ref():
    refimpl.build()
    if not refimpl.available():
        pytest.skip("oracle/_ref not built")
    return refimpl


def ofilter(orc, F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def small(cfg):
    return {1: lambda: WL.config1(n=64), 2: lambda: WL.config2(n=96),
            3: lambda: WL.config3(n=288, n_templates=2), 4: lambda: WL.config4(n=80),
            5: lambda: WL.config5(n=80, batch=2)}[cfg]()


def decompose(mod, w):
    group, args = w.decomp
    fn = mod.decompose_rotation2 if group == "rotation2" else mod.decompose_scale2
    return fn(w.filter_image, *args)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_decomposition_matches_reference(ref, orc, cfg):
    """freq_filter.hpp:63-129: ks and comps of the reference vs the oracle and
    vs the product's host decomposition (xc_decompose_*, host_filter.cpp)."""
    w = small(cfg)
    R = decompose(ref, w)
    O = decompose(orc, w)
    P = decompose(X, w)
    assert list(R.ks) == list(O.ks) == list(P.ks)
    assert rel(O.comps, R.comps) < 1e-13
    assert rel(P.comps, R.comps) < 1e-13


@pytest.mark.parametrize("cfg", [1, 2, 5])
def test_fast_paths_match_reference(ref, orc, cfg):
    w = small(cfg)
    R = decompose(ref, w)
    mode = 0 if w.mode == "xcorr" else 1
    H = w.signal[0].astype(np.float64)
    T = w.param[0].astype(np.float64)
    got, ops = ref.xfast(mode, H, 0, T, R)
    fn = orc.xcorr_fast if mode == 0 else orc.xconv_fast
    o, oops = fn(H, 0, T, ofilter(orc, R))[:2]
    assert ops == oops == len(R.ks)
    assert rel(o, got) < TIGHT


def test_scale_paths_and_smoothing_match_reference(ref, orc):
    w = small(4)
    R = decompose(ref, w)
    H = w.signal[0].astype(np.float64)
    S = w.param[0].astype(np.float64)
    OF = ofilter(orc, R)
    for mode, fn in ((0, orc.xcorr_fast), (1, orc.xconv_fast)):
        got, ops = ref.xfast(mode, H, 1, S, R)
        assert rel(fn(H, 1, S, OF)[0], got) < TIGHT
    out, ops, cl = ref.smooth_adaptive(H, 1, S, R)
    o, oops, ocl = orc.smooth_adaptive(H, 1, S, OF)
    assert ops == oops == 26 and cl == ocl
    assert rel(o, out) < TIGHT


def test_band_subset_periodic_and_errors_match_reference(ref, orc):
    w = small(1)
    R = decompose(ref, w)
    H = w.signal[0].astype(np.float64)[:40, :48]
    T = w.param[0].astype(np.float64)[:40, :48]
    OF = ofilter(orc, R)
    for comps in ([0], [-4, 1, 3]):
        for periodic in (False, True):
            got = ref.xcorr_fast(H, 0, T, R, comps, periodic)[0]
            assert rel(orc.xcorr_fast(H, 0, T, OF, comps, periodic)[0], got) < TIGHT
    with pytest.raises(ValueError, match="plan retains a component the filter lacks"):
        ref.xcorr_fast(H, 0, T, R, [99])
    S4 = small(4)
    R4 = decompose(ref, S4)
    bad = S4.param[0].astype(np.float64).copy()
    bad[3, 5] = 1e6
    with pytest.raises(ValueError) as e:
        ref.xcorr_fast(S4.signal[0], 1, bad, R4)
    with pytest.raises(ValueError) as eo:
        orc.xcorr_fast(S4.signal[0], 1, bad, ofilter(orc, R4))
    assert str(e.value) == str(eo.value) and "(5,3)" in str(e.value)


def test_filter2_fft_matches_reference(ref, orc):
    r = np.random.default_rng(3)
    for (h, w), (fh, fw), (cx, cy) in (((13, 9), (5, 5), (2, 2)), ((20, 31), (7, 3), (3, 1)),
                                       ((1, 9), (3, 3), (1, 1))):
        sig = r.normal(size=(h, w)) + 1j * r.normal(size=(h, w))
        f = r.normal(size=(fh, fw)) + 1j * r.normal(size=(fh, fw))
        for corr in (True, False):
            for per in (False, True):
                a = ref.filter2_fft(sig, f, cx, cy, corr, per)
                b = orc.filter2_fft(sig, f, cx, cy, corr, per)
                assert rel(b, a) < TIGHT
    assert all(ref.next_fast_size(n) == orc.next_fast_size(n) for n in range(1, 5000, 37))


def test_anglemax_peaks_match_reference(ref, orc):
    """Config 3 reduced: G_k of the reference (single-band xcorr_fast with a zero
    angle field, engine.hpp:300-319), the angle max, and find_peaks of the
    reference vs the oracle's band responses and find_peaks: same peak list."""
    w = small(3)
    R = decompose(ref, w)
    H = w.signal[0].astype(np.float64)
    zero = np.zeros_like(H)
    G = np.stack([ref.xcorr_fast(H, 0, zero, R, [int(k)])[0] for k in R.ks])
    Go = orc.band_responses(H, ofilter(orc, R), nthreads=4)
    assert rel(Go, G) < TIGHT
    score, arg = orc.anglemax(G, R.ks, 360)
    pk = ref.find_peaks(score, 32.0, 0.5)
    assert pk == orc.find_peaks(score, 32.0, 0.5)
    assert len(pk) >= 2
    for (cx, cy, _), (x, y, _) in zip(sorted(w.meta["truth"]), sorted(pk[:2])):
        assert abs(x - cx) <= 2 and abs(y - cy) <= 2


def test_detect_pattern_matches_reference(ref, orc):
    """vote_filter.hpp:83-91, 146-168: the reference's detection vs the oracle's."""
    r = np.random.default_rng(5)
    Rr = 8
    y, x = np.mgrid[-Rr:Rr + 1, -Rr:Rr + 1].astype(np.float64)
    pat = (np.exp(-((x - 3) ** 2 + (y + 2) ** 2) / 8.0) -
           0.8 * np.exp(-((x + 3) ** 2 + (y - 2) ** 2) / 6.0)) * np.exp(-(x * x + y * y) / 60.0)
    img = r.normal(0, 0.02, (96, 112))
    for cx, cy, a in ((30.0, 40.0, 0.4), (80.0, 60.0, 2.1)):
        WL.paste_rotated(img, pat, cx, cy, a)
    resp, pk, ops = ref.detect_pattern(pat, Rr, Rr, float(Rr), img, 16)
    wts, radius = orc.build_optimal_filter(pat, Rr, Rr, float(Rr))
    o = orc.detect_pattern(img, wts, radius, float(Rr), 16)
    assert ops == o[2]
    assert rel(o[0], resp) < TIGHT
    assert [(a, b) for a, b, _ in pk] == [(a, b) for a, b, _ in o[1]]
