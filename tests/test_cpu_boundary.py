"""CPU-side checks of the drop-in boundary (no GPU needed).

* the in-tree CUDA library loads and exports every symbol include/xconv_b200.h
  declares;
* the host-side filter logic behind the ABI (decomposition, rendering,
  reconstruction, inner DC, find_peaks, FFT planner) matches the oracle;
* without a CUDA device the hot path fails loudly (no CPU fallback).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "xconv_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(N.EXPORTS) == syms
    assert N.lib().xc_abi_version() == 2


def test_decomposition_matches_oracle(orc):
    rng = orc.Rng(11)
    R = 6
    filt = rng.random_smooth_filter(R)
    F = X.decompose_rotation2(filt, R, R, 16, 24, 64, R)
    O = orc.decompose_rotation2(filt, R, R, 16, 24, 64, R)
    assert np.array_equal(F.ks, O.ks)
    assert np.max(np.abs(F.comps - O.comps)) < 1e-14
    filt = rng.annular_filter(R)
    F = X.decompose_scale2(filt, R, R, 8, 48, 32, 1.0, R, R + 2.0)
    O = orc.decompose_scale2(filt, R, R, 8, 48, 32, 1.0, R, R + 2.0)
    assert np.max(np.abs(F.comps - O.comps)) < 1e-14
    assert abs(X.inner_dc_value(F) - orc.inner_dc_value(O)) < 1e-14
    for ci in range(F.n_components()):
        assert np.max(np.abs(X.render_component(F, ci, 13, 13, R, R) -
                             orc.render_component(O, ci, 13, 13, R, R))) < 1e-14
    assert np.max(np.abs(X.reconstruct(F, 13, 13, R, R, [-2, 0, 3]) -
                         orc.reconstruct(O, 13, 13, R, R, [-2, 0, 3]))) < 1e-14


def test_decomposition_errors_match_reference_text():
    f = np.zeros((9, 9))
    with pytest.raises(ValueError, match="n_angles must be >= 4 and even"):
        X.decompose_rotation2(f, 4, 4, 4, 8, 7, 4.0)
    with pytest.raises(ValueError, match="band limit too large for sampling rate"):
        X.decompose_rotation2(f, 4, 4, 40, 8, 16, 4.0)
    with pytest.raises(ValueError, match=r"r_min must be > 0 \(log-polar excludes the origin\)"):
        X.decompose_scale2(f, 4, 4, 4, 8, 16, 0.0, 4.0)
    with pytest.raises(ValueError, match="basis domain must reach the support radius"):
        X.decompose_scale2(f, 4, 4, 4, 8, 16, 0.5, 4.0, 3.0)
    with pytest.raises(ValueError, match="scale field must be strictly positive and finite"):
        X.XformField.scaling(np.array([[1.0, -1.0]]))


def test_find_peaks_matches_oracle(orc):
    r = np.random.default_rng(4)
    resp = np.round(r.standard_normal((40, 50)), 1)  # many exact ties
    got = [(p.x, p.y, p.value) for p in X.find_peaks(resp, 2.5, 0.3)]
    assert got == orc.find_peaks(resp, 2.5, 0.3)
    got32 = X.find_peaks(resp.astype(np.float32), 3.0, 0.5)
    assert [(p.x, p.y) for p in got32] == [(p[0], p[1]) for p in
                                           orc.find_peaks(resp.astype(np.float32), 3.0, 0.5)]


def test_hot_path_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    F = X.decompose_rotation2(np.ones((5, 5)), 2, 2, 2, 4, 8, 2.0)
    with pytest.raises(RuntimeError):
        X.xcorr_fast(np.zeros((4, 4)), X.XformField.rotation(np.zeros((4, 4))), F)


def test_fft_planner_pad_rule(orc):
    # pads are the smallest plannable 2/3/5-smooth length >= extent + R; for
    # the BASELINE configs this equals the reference's next_fast_size(H + 2R + 1)
    import ctypes
    assert orc.next_fast_size(256 + 31) == 288 and orc.next_fast_size(4096 + 63) == 4320


def test_pad_rule_and_tile_count_host_logic():
    """api.cu pick_pad2d / tile_count (host logic, no GPU): the pad is a planned
    length >= the request; the BASELINE configs keep their pads; requests between
    two pair-plan lengths take the next one; axes beyond 4320 - R split into
    balanced halo tiles whose padded extent fits the longest plan."""
    L = N.lib()
    pair = [288, 576, 768, 1024, 1152, 1280, 1536, 1920, 2048, 2160, 2304, 2560, 2880, 3072,
            3456, 4096, 4320]
    # config 1: 256 + 15, config 2: 1024 + 16, config 4: 2048 + 32, configs 3 / 5: 4096 + 32 / 31
    for n, pad in [(271, 288), (1040, 1152), (2080, 2160), (4128, 4320), (4127, 4320)]:
        assert L.xc_debug_pick_pad(n) == pad
    for n in list(range(1, 400, 7)) + list(range(400, 4321, 53)) + pair:
        p = L.xc_debug_pick_pad(n)
        assert p >= n
        if n >= 289:  # from here on a pair plan is always the cheapest candidate
            assert p == min(q for q in pair if q >= n), (n, p)
    for n in (5, 16, 33):  # tiny requests keep a small length (no inflation to 288)
        assert L.xc_debug_pick_pad(n) < 128
    assert L.xc_debug_pick_pad(6000) >= 6000  # beyond the plans: a generic smooth length
    # tiles
    for R in (0, 9, 31, 100):
        for n in (1, 4000, 4320 - R, 4321 - R, 8192, 20000):
            t = L.xc_debug_tile_count(n, R)
            assert t >= 1
            if n + R <= 4320:
                assert t == 1
            else:
                interior = -(-n // t)
                assert interior + 3 * R <= 4320  # halo both sides + the pad's R
                assert t == 1 or -(-n // (t - 1)) + 3 * R > 4320  # and no fewer tiles would do
