"""Line integral convolution over the GPU path (lic.hpp:9-55):
seeded white noise smeared along a rotation field by the extended convolution
with a rotating anisotropic Gaussian.  The normalized form is
smooth_adaptive (engine.hpp:385-419); the unnormalized form is the real part
of xconv_fast (engine.hpp:331-373).  Noise and kernel are host work, once per
call, as in the reference; the band filtering and steering run on the GPU."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .engine import XformField, XformKind, decompose_rotation2, smooth_adaptive, xconv_fast


def white_noise(width: int, height: int, seed: int) -> np.ndarray:
    """lic.hpp:9-17: std::mt19937_64(seed), (rng() >> 11) * 2^-53 per pixel in
    y-major order; returned as a [height][width] float64 array (bit-identical
    for a given seed)."""
    out = np.zeros((int(height), int(width)), np.float64)
    N.check(N.lib().xc_white_noise(C.c_ulonglong(int(seed) & (2**64 - 1)), int(height),
                                   int(width), N.XC_ROW_MAJOR,
                                   out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def anisotropic_gaussian(length: float, width: float) -> np.ndarray:
    """lic.hpp:20-32: exp(-x^2/(2 length^2) - y^2/(2 width^2)) on the disc of
    radius R = ceil(2.5 length), (2R+1)^2 grid centred at (R, R), oriented
    along +x."""
    R = int(math.ceil(2.5 * length))
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    f = np.exp(-x * x / (2 * length * length) - y * y / (2 * width * width))
    f[x * x + y * y > float(R) * R] = 0.0
    return f


def lic(field: XformField, length: float, width: float, seed: int, normalized: bool = True,
        K: int = 16) -> np.ndarray:
    """lic.hpp:37-55.  Returns the [height][width] float64 image."""
    if field.kind != XformKind.rotation2:
        raise ValueError("lic needs a rotation2 field")
    if not (length > width) or not (width > 0):
        raise ValueError("need length > width > 0")
    h, w = np.asarray(field.values).shape
    noise = white_noise(w, h, seed)
    kern = anisotropic_gaussian(length, width)
    R = (kern.shape[1] - 1) // 2
    n_angles = max(64, 4 * int(K))
    F = decompose_rotation2(kern, float(R), float(R), int(K), max(8, R), n_angles, R + 0.5,
                            device=True)  # a per-call filter build, on the GPU
    if normalized:
        return np.asarray(smooth_adaptive(noise, field, F).output, np.float64)
    return np.asarray(xconv_fast(noise, field, F).output.real, np.float64)
