"""Filter decomposition on the GPU (freq_filter.hpp:63-129,
polar.hpp:46-83): xc_decompose_rotation2_device / xc_decompose_scale2_device
against the REFERENCE itself (oracle/_ref, its headers compiled unchanged) and
against the product's host decomposition, on every BASELINE config's filter
and on edge cases (Nyquist split, off-centre origin, samples outside the
image, the scale group's basis domain).  Both sides are fp64; the device
evaluates the band phases with sincospi of an exact quotient and the polar
angles with the device cos/sin, so the bound is 1e-12 relative L2 (the host
decompositions agree with the reference to 1e-13, tests/test_ref_parity.py).
Also the per-call users: detect_pattern (decomposes its vote filter on the
device) and match_contours / lic (device=True) are covered by their own tests.
"""
import numpy as np
import pytest

import paper_2006_13188_b200 as X
from oracle import refimpl
from paper_2006_13188_b200 import workloads as WL

pytestmark = pytest.mark.gpu
TIGHT = 1e-12


@pytest.fixture(scope="module")
def ref():
    refimpl.build()
    assert refimpl.available(), "oracle/_ref missing: build it with `make -C oracle ref`"
    return refimpl


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def both(mod_fn, x_fn, img, *args):
    return mod_fn(img, *args), x_fn(img, *args, device=True), x_fn(img, *args)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_device_decomposition_matches_reference(ref, cfg):
    # the filters are the full-size ones; only the images are reduced
    w = {1: lambda: WL.config1(n=64), 2: lambda: WL.config2(n=96),
         3: lambda: WL.config3(n=288, n_templates=2), 4: lambda: WL.config4(n=80),
         5: lambda: WL.config5(n=80, batch=1)}[cfg]()
    group, args = w.decomp
    name = "decompose_rotation2" if group == "rotation2" else "decompose_scale2"
    R, D, H = both(getattr(ref, name), getattr(X, name), w.filter_image, *args)
    assert list(R.ks) == list(D.ks) == list(H.ks)
    assert rel(D.comps, R.comps) < TIGHT
    assert rel(D.comps, H.comps) < TIGHT


@pytest.mark.parametrize("n_angles,K", [(16, 16), (32, 8), (66, 64)])
def test_device_rotation_nyquist_and_offcentre(ref, n_angles, K):
    """|k| = n_angles / 2 is halved (split over +-k); an off-centre origin and
    a radius past the image edge sample zeros (field.hpp:51-62)."""
    rng = np.random.default_rng(7)
    img = rng.standard_normal((21, 17)) + 1j * rng.standard_normal((21, 17))
    for cx, cy, r_max in [(8.0, 10.0, 8.0), (3.3, 15.7, 12.5)]:
        R, D, H = both(ref.decompose_rotation2, X.decompose_rotation2, img, cx, cy, K, 9,
                       n_angles, r_max)
        assert list(R.ks) == list(D.ks)
        assert rel(D.comps, R.comps) < TIGHT
        assert rel(D.comps, H.comps) < TIGHT


def test_device_scale_with_basis_domain(ref):
    rng = np.random.default_rng(8)
    img = rng.random((33, 33)).astype(np.complex128)
    for r_domain in (0.0, 24.0):
        R, D, H = both(ref.decompose_scale2, X.decompose_scale2, img, 16.0, 16.0, 10, 24, 32,
                       1.0, 16.0, r_domain)
        assert list(R.ks) == list(D.ks)
        assert rel(D.comps, R.comps) < TIGHT
        assert D.r_domain == H.r_domain


def test_device_decomposition_errors_match_host():
    img = np.ones((9, 9), np.complex128)
    cases = [
        (X.decompose_rotation2, (img, 4.0, 4.0, 8, 0, 16, 4.0)),    # n_radii
        (X.decompose_rotation2, (img, 4.0, 4.0, 8, 4, 6 + 1, 4.0)),  # odd n_angles
        (X.decompose_rotation2, (img, 4.0, 4.0, 40, 4, 16, 4.0)),   # band limit
        (X.decompose_scale2, (img, 4.0, 4.0, 4, 8, 16, 0.0, 4.0)),  # r_min
        (X.decompose_scale2, (img, 4.0, 4.0, 4, 8, 16, 1.0, 4.0, 2.0)),  # domain
    ]
    for fn, args in cases:
        with pytest.raises(ValueError) as host:
            fn(*args)
        with pytest.raises(ValueError) as dev:
            fn(*args, device=True)
        assert str(host.value) == str(dev.value)


def test_device_filter_drives_the_pipeline_like_the_host_filter(orc):
    """A device-decomposed filter gives the same xconv_fast output as the host
    one (config 2's filter, reduced image)."""
    w = WL.config2(n=96)
    group, args = w.decomp
    Fd = X.decompose_rotation2(w.filter_image, *args, device=True)
    T = X.XformField.rotation(w.param[0])
    a = X.xconv_fast(w.signal[0], T, Fd).output
    b = X.xconv_fast(w.signal[0], T, w.filt).output
    assert rel(a, b) < 1e-6
