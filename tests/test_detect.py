"""Pattern detection: vote filters on the host, detect_pattern
on the GPU (gradient kernel + the scatter pipeline + NMS), against the oracle's
restatement of vote_filter.hpp and the reference's own detection tests
(proj/tests/test_detect.cpp)."""
import math

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from paper_2006_13188_b200.workloads import paste_rotated


def bump_pattern(R):
    """test_detect.cpp:11-31: asymmetric Gaussian bumps under an envelope."""
    bumps = [(-2.5, 0.5, 1.0, 1.6), (2.0, -2.0, -0.8, 1.3), (1.0, 3.0, 0.6, 1.8),
             (-1.0, -3.0, 0.9, 1.2)]
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    v = np.zeros_like(x)
    for bx, by, a, s in bumps:
        v += a * np.exp(-((x - bx) ** 2 + (y - by) ** 2) / (2 * s * s))
    env = 0.38 * R
    return v * np.exp(-(x * x + y * y) / (2 * env * env))


def rot90(f):
    """test_detect.cpp:55-61: new(x, y) = old(y, W-1-x)."""
    h, w = f.shape
    out = np.zeros((w, h))
    for y in range(w):
        for x in range(h):
            out[y, x] = f[w - 1 - x, y]
    return out


# ------------------------------------------------------------- host (CPU)

@pytest.mark.parametrize("R,nearest", [(6, False), (8, False), (8, True), (11, False)])
def test_optimal_filter_matches_oracle(orc, R, nearest):  # vote_filter.hpp:62-91
    pat = bump_pattern(R)
    vf = X.build_optimal_filter(pat, R, R, float(R), nearest)
    w, r = orc.build_optimal_filter(pat, R, R, float(R), nearest)
    assert vf.radius == r and np.array_equal(vf.weights, w)
    # off-centre support radius
    vf2 = X.build_optimal_filter(pat, R - 1.5, R + 0.5, R - 0.5, nearest)
    w2, _ = orc.build_optimal_filter(pat, R - 1.5, R + 0.5, R - 0.5, nearest)
    assert np.array_equal(vf2.weights, w2)


def test_vote_filter_matches_oracle_and_mass(orc):  # test_detect.cpp:199-214
    R = 7
    pat = bump_pattern(R)
    vf = X.build_optimal_filter(pat, R, R, float(R))
    mag, _ = orc.gradient(pat)
    y, x = np.mgrid[0:pat.shape[0], 0:pat.shape[1]]
    inside = (x - R) ** 2 + (y - R) ** 2 <= R * R
    assert abs(vf.total_mass() - mag[inside].sum()) < 1e-9 * mag[inside].sum()
    rng = np.random.default_rng(3)
    weight = rng.uniform(0, 1, (20, 17))
    frame = rng.uniform(-np.pi, np.pi, (20, 17))
    a = X.build_vote_filter(weight, frame, 8.3, 9.6, 6.5)
    b, r = orc.build_vote_filter(weight, frame, 8.3, 9.6, 6.5)
    assert a.radius == r and np.array_equal(a.weights, b)


def test_vote_filter_errors():  # vote_filter.hpp:66, 79, 87
    pat = bump_pattern(5)
    with pytest.raises(ValueError, match="support radius must be > 0"):
        X.build_optimal_filter(pat, 5, 5, 0.0)
    with pytest.raises(ValueError, match="center must lie inside the pattern"):
        X.build_optimal_filter(pat, -1, 5, 3.0)
    with pytest.raises(ValueError, match="degenerate pattern: no votes in support"):
        X.build_optimal_filter(np.zeros((11, 11)), 5, 5, 3.0)


# ------------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_three_pasted_rotations_found(orc):  # test_detect.cpp:75-108
    n, R = 96, 8
    pat = bump_pattern(R)
    img = np.zeros((n, n))
    truth = [(24, 26, 0.0), (70, 25, math.pi / 2), (30, 70, 37.0 * math.pi / 180)]
    for cx, cy, a in truth:
        paste_rotated(img, pat, cx, cy, a)
    vf = X.build_optimal_filter(pat, R, R, float(R))
    det = X.detect_pattern(img, vf, 16)
    assert len(det.peaks) >= 3
    used = [False] * 3
    for p in det.peaks[:3]:
        for t, (cx, cy, _) in enumerate(truth):
            if not used[t] and math.hypot(p.x - cx, p.y - cy) <= 2.0:
                used[t] = True
                break
    assert all(used)
    strong = 0.7 * det.peaks[0].value
    for p in det.peaks:
        if p.value >= strong:
            assert min(math.hypot(p.x - cx, p.y - cy) for cx, cy, _ in truth) <= 2.0
    # parity with the oracle's detect_pattern (double) on the same image
    resp, opk, ops = orc.detect_pattern(img, vf.weights, vf.radius, vf.eps, 16)
    assert det.standard_ops == ops
    assert orc.rel_l2(det.response, resp) < 1e-5
    assert [(p.x, p.y) for p in det.peaks[:3]] == [(x, y) for x, y, _ in opk[:3]]


@pytest.mark.gpu
def test_blank_image_gives_zero_response():  # test_detect.cpp:110-117
    R = 6
    vf = X.build_optimal_filter(bump_pattern(R), R, R, float(R))
    det = X.detect_pattern(np.zeros((32, 32)), vf, 8)
    assert np.max(np.abs(det.response)) < 1e-12


@pytest.mark.gpu
def test_response_error_monotone_in_band_limit(orc):  # test_detect.cpp:119-135
    n, R = 64, 8
    pat = bump_pattern(R)
    img = np.zeros((n, n))
    paste_rotated(img, pat, 22, 25, 0.4)
    paste_rotated(img, pat, 44, 40, 2.1)
    vf = X.build_optimal_filter(pat, R, R, float(R))
    na = 64
    full = X.detect_pattern(img, vf, na, 0, na).response
    prev = np.inf
    for K in (2, 4, 8, 16):
        det = X.detect_pattern(img, vf, K, 0, na)
        err = orc.rel_l2(det.response, full)
        assert err <= prev + 1e-6  # fp32 response (reference: 1e-12 in double)
        prev = err
        ref = orc.detect_pattern(img, vf.weights, vf.radius, vf.eps, K, 0, na)[0]
        assert orc.rel_l2(det.response, ref) < 1e-5


@pytest.mark.gpu
def test_peaks_covariant_with_rot90():  # test_detect.cpp:137-159
    n, R = 64, 8
    pat = bump_pattern(R)
    img = np.zeros((n, n))
    paste_rotated(img, pat, 24, 20, 0.7)
    paste_rotated(img, pat, 42, 44, 2.9)
    vf = X.build_optimal_filter(pat, R, R, float(R))
    det = X.detect_pattern(img, vf, 16)
    det_r = X.detect_pattern(rot90(img), vf, 16)
    assert len(det.peaks) >= 2 and len(det_r.peaks) >= 2
    for p in det.peaks[:2]:
        ex, ey = n - 1 - p.y, p.x
        assert min(math.hypot(q.x - ex, q.y - ey) for q in det_r.peaks[:2]) <= 1.0


@pytest.mark.gpu
def test_self_response_peaks_at_center():  # test_detect.cpp:161-168
    R = 8
    pat = bump_pattern(R)
    vf = X.build_optimal_filter(pat, R, R, float(R))
    det = X.detect_pattern(pat, vf, 32)
    assert det.peaks and math.hypot(det.peaks[0].x - R, det.peaks[0].y - R) <= 1.0


@pytest.mark.gpu
def test_detect_float32_image_and_errors(orc):
    n, R = 48, 6
    pat = bump_pattern(R)
    img = np.zeros((n, n))
    paste_rotated(img, pat, 20, 23, 1.1)
    vf = X.build_optimal_filter(pat, R, R, float(R))
    d32 = X.detect_pattern(img.astype(np.float32), vf, 12)
    assert d32.response.dtype == np.float32
    ref = orc.detect_pattern(img.astype(np.float32).astype(np.float64), vf.weights, vf.radius,
                             vf.eps, 12)[0]
    assert orc.rel_l2(d32.response, ref) < 1e-5
    with pytest.raises(ValueError, match="K must be >= 1"):
        X.detect_pattern(img, vf, 0)
    with pytest.raises(ValueError, match="gradient requires real field"):
        X.detect_pattern(img.astype(np.complex128), vf, 8)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_find_peaks_device_equals_host(orc, dtype):  # vote_filter.hpp:107-134
    r = np.random.default_rng(21)
    resp = np.round(r.uniform(-1, 1, (131, 97)) * 8) / 8  # many exact ties
    resp = resp.astype(dtype)
    for radius, frac in [(2.5, 0.3), (1.0, 0.0), (4.0, 0.6), (0.5, 0.5)]:
        host = [(p.x, p.y, p.value) for p in X.find_peaks(resp, radius, frac)]
        dev = [(p.x, p.y, p.value) for p in X.find_peaks(resp, radius, frac, gpu=True)]
        assert dev == host
        assert host == orc.find_peaks(resp.astype(np.float64), radius, frac)
