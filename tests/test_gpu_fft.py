"""Standalone GPU FFT parity (fft.hpp:20-53):
xc_fft2 runs the pipeline's own row (F1) and column (F2) transforms -- the pair
engine at 1152 / 2160 / 4320, the fast and generic kernels elsewhere -- on a
complex grid.  Against numpy's double-precision FFT at relative L2 <= 1e-6
(fp32 transforms of O(1) data), against the reference's own fft2 (oracle/_ref,
Eigen's kissfft through the shim) on small grids, forward unscaled and inverse
scaled 1/n, with odd widths (run as the transposed problem) and round trips.
"""
import numpy as np
import pytest

import paper_2006_13188_b200 as X
from oracle import refimpl

pytestmark = pytest.mark.gpu
TOL = 1e-6


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def grid(h, w, seed=0, dtype=np.complex64):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((h, w)) + 1j * rng.standard_normal((h, w))).astype(dtype)


@pytest.mark.parametrize("n", [288, 1080, 1152, 2160, 4320])
def test_square_sizes_match_numpy(n):
    x = grid(n, n, n)
    ref = np.fft.fft2(x.astype(np.complex128))
    got = X.fft2(x)
    assert got.dtype == np.complex64
    assert rel(got, ref) < TOL, rel(got, ref)
    back = X.fft2(ref.astype(np.complex64), inverse=True)
    assert rel(back, x) < TOL


@pytest.mark.parametrize("h,w", [(96, 160), (1152, 2160), (4320, 1080), (36, 64), (64, 45),
                                 (2, 2), (1, 8), (8, 1)])
def test_rectangular_and_odd_extents(h, w):
    x = grid(h, w, h * 7 + w, np.complex128)
    got = X.fft2(x)
    assert got.dtype == np.complex128
    assert rel(got, np.fft.fft2(x)) < TOL
    assert rel(X.fft2(x, inverse=True), np.fft.ifft2(x)) < TOL


def test_matches_the_reference_fft2():
    refimpl.build()
    assert refimpl.available()
    for h, w in [(30, 48), (60, 90), (288, 288)]:
        x = grid(h, w, h + w, np.complex128)
        for inv in (False, True):
            assert rel(X.fft2(x, inverse=inv), refimpl.fft2(x, inv)) < TOL


def test_validation():
    with pytest.raises(ValueError, match="one even extent"):
        X.fft2(np.zeros((3, 5), np.complex64))
    with pytest.raises(ValueError):
        X.fft2(np.zeros((4, 4, 4), np.complex64))
    with pytest.raises(ValueError, match="unsupported transform length"):
        X.fft2(np.zeros((37, 64), np.complex64))  # not 2,3,5-smooth
