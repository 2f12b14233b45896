"""Seeded synthetic inputs for the BASELINE.json configurations.

Input generation only (numpy/scipy on the host): these arrays are what both
the B200 path and the CPU oracle consume.  The reference publishes no
datasets for this path; the configs are synthetic by definition (BASELINE.json
`configs`).  Gap decisions recorded in DESIGN.md ("Workloads"):

  * complex coefficients "~N(0,1)": real and imaginary parts each N(0,1);
  * config 3 template: smooth random bumps under an envelope
    (proj/tests/helpers.hpp:40-64 style), pasted with bilinear rotation
    (acceptance.cpp:138-150 paste_rotated);
  * config 4: Gaussian filter sigma = 8 px truncated at r = 32, K = 12 ->
    13 log-radial bands (an odd count is forced by freq_filter.hpp:52-59),
    r_min = 1; s = 8**z with z a blurred (sigma 16) noise field rescaled to
    [0, 1];
  * config 5 uses n_angles = 130 so |k| = 32 is not a Nyquist-split band.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy import ndimage

from .engine import FreqFilter2, decompose_rotation2, decompose_scale2


def gaussian_blur(img: np.ndarray, sigma: float) -> np.ndarray:
    """Separable normalized Gaussian, radius ceil(3 sigma), zero boundary
    (contour.hpp:28-55)."""
    R = max(1, int(math.ceil(3 * sigma)))
    k = np.exp(-np.arange(-R, R + 1) ** 2 / (2 * sigma * sigma))
    k /= k.sum()
    t = ndimage.correlate1d(img.astype(np.float64), k, axis=1, mode="constant")
    return ndimage.correlate1d(t, k, axis=0, mode="constant")


def gradient(img: np.ndarray):
    """Central differences, one-sided at the borders; direction 0 where the
    magnitude vanishes (field.hpp:202-237)."""
    gy, gx = np.gradient(img.astype(np.float64))
    mag = np.hypot(gx, gy)
    return mag, np.where(mag > 0, np.arctan2(gy, gx), 0.0)


def angular_filter(R: int, sigma: float, m_max: int, rng: np.random.Generator) -> np.ndarray:
    """(2R+1)^2 filter: Gaussian radial window x random angular profile
    band-limited to |m| <= m_max, complex N(0,1) coefficients (y points down)."""
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    phi = np.arctan2(y, x)
    c = rng.standard_normal(2 * m_max + 1) + 1j * rng.standard_normal(2 * m_max + 1)
    prof = sum(c[m + m_max] * np.exp(1j * m * phi) for m in range(-m_max, m_max + 1))
    return np.exp(-(x * x + y * y) / (2 * sigma * sigma)) * prof


def smooth_template(size: int, rng: np.random.Generator, n_bumps: int = 8) -> np.ndarray:
    """size x size real template of Gaussian bumps under a radial envelope."""
    c = (size - 1) / 2.0
    y, x = np.mgrid[0:size, 0:size].astype(np.float64)
    v = np.zeros((size, size))
    for _ in range(n_bumps):
        bx, by = rng.uniform(-0.5, 0.5, 2) * c
        a = rng.uniform(-1, 1)
        s = (0.08 + 0.06 * rng.uniform()) * size
        v += a * np.exp(-((x - c - bx) ** 2 + (y - c - by) ** 2) / (2 * s * s))
    env = 0.38 * size
    return v * np.exp(-((x - c) ** 2 + (y - c) ** 2) / (2 * env * env))


def paste_rotated(img: np.ndarray, pat: np.ndarray, cx: float, cy: float, angle: float):
    """Add `pat` rotated by `angle` about (cx, cy) with bilinear sampling
    (acceptance.cpp:138-150)."""
    S = pat.shape[0]
    pc = (S - 1) / 2.0
    c, s = math.cos(-angle), math.sin(-angle)
    r = int(math.ceil(pc)) + 1
    x0, y0 = int(round(cx)), int(round(cy))
    ys, xs = np.mgrid[y0 - r:y0 + r + 1, x0 - r:x0 + r + 1]
    ok = (xs >= 0) & (ys >= 0) & (xs < img.shape[1]) & (ys < img.shape[0])
    ox, oy = xs - cx, ys - cy
    sx, sy = c * ox - s * oy + pc, s * ox + c * oy + pc
    fx, fy = np.floor(sx), np.floor(sy)
    tx, ty = sx - fx, sy - fy
    fx, fy = fx.astype(int), fy.astype(int)

    def tap(xi, yi):
        inside = (xi >= 0) & (yi >= 0) & (xi < S) & (yi < S)
        return np.where(inside, pat[np.clip(yi, 0, S - 1), np.clip(xi, 0, S - 1)], 0.0)

    val = ((1 - ty) * ((1 - tx) * tap(fx, fy) + tx * tap(fx + 1, fy)) +
           ty * ((1 - tx) * tap(fx, fy + 1) + tx * tap(fx + 1, fy + 1)))
    img[ys[ok], xs[ok]] += val[ok]


@dataclass
class Workload:
    name: str
    mode: str                    # "xcorr" | "xconv" | "smooth" | "anglemax"
    signal: np.ndarray           # (B, H, W) float32
    param: np.ndarray | None     # (B, H, W) float32 angle or scale, or None
    kind: int                    # XformKind
    filt: FreqFilter2
    filter_image: np.ndarray
    meta: dict = field(default_factory=dict)
    # how `filt` was decomposed from `filter_image`: ("rotation2", (cx, cy, K,
    # n_radii, n_angles, r_max)) or ("scale2", (cx, cy, K, n_radii, n_angles,
    # r_min, r_max)) -- lets tests and the reference arm rebuild it with the
    # oracle or the reference itself
    decomp: tuple = ()

    @property
    def bands(self) -> int:
        return self.filt.n_components()

    def units(self) -> int:
        """work units = H * W * standard_ops * images (engine.hpp:318/367/406)."""
        B, H, W = self.signal.shape
        ops = self.bands * (2 if self.mode == "smooth" else 1)
        return B * H * W * ops


def _decompose(D, f, backend):
    """Decompose the filter image with the product's host code (default) or a
    test-side backend module (oracle.oracle / oracle.refimpl: the bench's
    reference arm builds its filter without loading the product library)."""
    import sys
    mod = backend if backend is not None else sys.modules[__name__]
    fn = mod.decompose_rotation2 if D[0] == "rotation2" else mod.decompose_scale2
    return fn(f, *D[1])


def config1(n: int = 256, seed: int = 0, backend=None) -> Workload:
    rng = np.random.default_rng([seed, 1])
    sig = rng.uniform(0, 1, (1, n, n)).astype(np.float32)
    th = rng.uniform(0, 2 * math.pi, (1, n, n)).astype(np.float32)
    f = angular_filter(15, 6.0, 4, rng)
    D = ("rotation2", (15, 15, 8, 30, 32, 15.0))
    F = _decompose(D, f, backend)
    return Workload(f"cfg1-xcorr-rot-{n}", "xcorr", sig, th, 0, F, f, decomp=D)


def config2(n: int = 1024, seed: int = 0, backend=None) -> Workload:
    rng = np.random.default_rng([seed, 2])
    sig = rng.uniform(0, 1, (1, n, n)).astype(np.float32)
    _, d = gradient(gaussian_blur(rng.standard_normal((n, n)), 4.0))
    th = d[None].astype(np.float32)
    f = angular_filter(16, 8.0, 8, rng)
    D = ("rotation2", (16, 16, 16, 32, 34, 16.0))
    F = _decompose(D, f, backend)
    return Workload(f"cfg2-xconv-rot-{n}", "xconv", sig, th, 0, F, f, decomp=D)


def config3(n: int = 4096, n_templates: int = 3, seed: int = 0, backend=None) -> Workload:
    rng = np.random.default_rng([seed, 3])
    img = rng.standard_normal((n, n))
    tpl = smooth_template(64, rng)
    truth = []
    margin = min(80, n // 4)
    sep = min(160, n // 2)
    for _ in range(n_templates):
        while True:
            cx, cy = rng.uniform(margin, n - margin, 2)
            if all(math.hypot(cx - a, cy - b) > sep for a, b, _ in truth):
                break
        ang = rng.uniform(0, 2 * math.pi)
        paste_rotated(img, 4.0 * tpl, cx, cy, ang)
        truth.append((cx, cy, ang))
    D = ("rotation2", (31.5, 31.5, 32, 64, 66, 31.5))
    F = _decompose(D, tpl, backend)
    return Workload(f"cfg3-anglemax-rot-{n}", "anglemax", img[None].astype(np.float32), None,
                    0, F, tpl, {"truth": truth, "n_angles": 360, "nms_radius": 32.0,
                                "threshold": 0.5}, decomp=D)


def config4(n: int = 2048, seed: int = 0, backend=None) -> Workload:
    rng = np.random.default_rng([seed, 4])
    sig = (rng.uniform(0, 1, (n, n)) + rng.normal(0, 0.05, (n, n)))[None].astype(np.float32)
    z = gaussian_blur(rng.standard_normal((n, n)), 16.0)
    z = (z - z.min()) / max(z.max() - z.min(), 1e-300)
    s = (8.0 ** z)[None].astype(np.float32)
    R = 32
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    f = np.exp(-(x * x + y * y) / (2 * 8.0 ** 2))
    f[x * x + y * y > R * R] = 0
    D = ("scale2", (R, R, 12, 64, 32, 1.0, float(R)))
    F = _decompose(D, f, backend)
    return Workload(f"cfg4-smooth-scale-{n}", "smooth", sig, s, 1, F, f, decomp=D)


def config5(n: int = 4096, batch: int = 16, seed: int = 0, backend=None) -> Workload:
    rng = np.random.default_rng([seed, 5])
    sig = rng.uniform(0, 1, (batch, n, n)).astype(np.float32)
    th = rng.uniform(0, 2 * math.pi, (batch, n, n)).astype(np.float32)
    f = angular_filter(31, 14.0, 32, rng)
    D = ("rotation2", (31, 31, 64, 62, 130, 31.0))
    F = _decompose(D, f, backend)
    return Workload(f"cfg5-xcorr-rot-{batch}x{n}", "xcorr", sig, th, 0, F, f, decomp=D)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
