"""Contour (fragment) matching over the GPU path (contour.hpp:8-189; SURVEY
8(b) caller `match_contours`, contour.hpp:168): the complement filter is built
from the query scene with negated normals, scattered over the target by
xconv_fast on the GPU, and the top peaks are refined by a 1D angular search on
polar patches.  Rasterization, the vote filter, the decomposition and the
refinement are host work, as in the reference."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .engine import (XformField, build_vote_filter, decompose_rotation2, find_peaks,
                     xconv_fast)


def normalize_angle(a):
    """field.hpp:122-127: [-pi, pi)."""
    a = np.fmod(np.asarray(a, np.float64) + math.pi, 2 * math.pi)
    a = np.where(a < 0, a + 2 * math.pi, a)
    return a - math.pi


def gaussian_blur(img: np.ndarray, sigma: float) -> np.ndarray:
    """contour.hpp:29-55: separable normalized Gaussian, radius max(1, ceil(3
    sigma)), zero outside the grid (x pass, then y pass)."""
    R = max(1, int(math.ceil(3 * sigma)))
    i = np.arange(-R, R + 1, dtype=np.float64)
    k = np.exp(-(i * i) / (2 * sigma * sigma))
    k /= k.sum()
    a = np.asarray(img, np.float64)
    h, w = a.shape
    tmp = np.zeros_like(a)
    for d in range(-R, R + 1):
        lo, hi = max(0, -d), min(w, w - d)
        if lo < hi:
            tmp[:, lo:hi] += k[d + R] * a[:, lo + d:hi + d]
    out = np.zeros_like(a)
    for d in range(-R, R + 1):
        lo, hi = max(0, -d), min(h, h - d)
        if lo < hi:
            out[lo:hi, :] += k[d + R] * tmp[lo + d:hi + d, :]
    return out


@dataclass
class ContourScene:  # contour.hpp:13-22
    signal: np.ndarray        # [height][width] >= 0
    normal_angle: np.ndarray  # radians
    coverage: np.ndarray      # smoothed magnitude of the normal vector field
    sigma: float = 1.5

    @property
    def width(self) -> int:
        return self.signal.shape[1]

    @property
    def height(self) -> int:
        return self.signal.shape[0]


@dataclass
class ContourMatch:  # contour.hpp:109-113
    x: int
    y: int
    angle: float
    score: float


def _lround(v: float) -> int:
    """std::lround: halves away from zero."""
    return int(math.copysign(math.floor(abs(v) + 0.5), v))


def rasterize_contours(lines, width: int, height: int, sigma: float = 1.5) -> ContourScene:
    """contour.hpp:62-106: unit stamping of each segment (lround of the
    parametric points, ceil(len) steps) with its left-hand normal accumulated,
    then all three grids blurred."""
    sig = np.zeros((height, width))
    nxs = np.zeros((height, width))
    nys = np.zeros((height, width))
    for line in lines:
        pts = [(float(p[0]), float(p[1])) for p in line]
        for (ax, ay), (bx, by) in zip(pts[:-1], pts[1:]):
            ln = math.hypot(bx - ax, by - ay)
            if ln == 0.0:
                continue
            dx, dy = (bx - ax) / ln, (by - ay) / ln
            nx, ny = dy, -dx
            steps = max(1, int(math.ceil(ln)))
            for s in range(steps + 1):
                t = s / steps
                x, y = _lround(ax + t * (bx - ax)), _lround(ay + t * (by - ay))
                if x < 0 or y < 0 or x >= width or y >= height:
                    continue
                sig[y, x] = 1.0
                nxs[y, x] += nx
                nys[y, x] += ny
    ssig = gaussian_blur(sig, sigma)
    snx = gaussian_blur(nxs, sigma)
    sny = gaussian_blur(nys, sigma)
    cov = np.sqrt(snx * snx + sny * sny)
    ang = np.where(cov > 0, np.arctan2(sny, snx), 0.0)
    return ContourScene(ssig, ang, cov, sigma)


def _sample(f: np.ndarray, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """field.hpp:52-62: bilinear, zero outside the grid."""
    h, w = f.shape
    fx, fy = np.floor(x), np.floor(y)
    x0, y0 = fx.astype(np.int64), fy.astype(np.int64)
    tx, ty = x - fx, y - fy

    def tap(xi, yi):
        ok = (xi >= 0) & (yi >= 0) & (xi < w) & (yi < h)
        return np.where(ok, f[np.clip(yi, 0, h - 1), np.clip(xi, 0, w - 1)], 0.0)

    return ((1 - ty) * ((1 - tx) * tap(x0, y0) + tx * tap(x0 + 1, y0)) +
            ty * ((1 - tx) * tap(x0, y0 + 1) + tx * tap(x0 + 1, y0 + 1)))


def resample_polar(f: np.ndarray, cx: float, cy: float, n_radii: int, n_angles: int,
                   r_max: float) -> np.ndarray:
    """polar.hpp:46-61: (n_radii, n_angles) samples at r_j = (j + 0.5) r_max /
    n_radii, theta_m = 2 pi m / n_angles."""
    if n_radii < 1:
        raise ValueError("n_radii must be >= 1")
    if n_angles < 4 or n_angles % 2 != 0:
        raise ValueError("n_angles must be >= 4 and even")
    if not r_max > 0:
        raise ValueError("r_max must be > 0")
    r = (np.arange(n_radii) + 0.5) * r_max / n_radii
    th = 2 * math.pi * np.arange(n_angles) / n_angles
    return _sample(np.asarray(f, np.float64), cx + r[:, None] * np.cos(th)[None, :],
                   cy + r[:, None] * np.sin(th)[None, :])


def _polar_sample(g: np.ndarray, r_max: float, r: float, theta: np.ndarray) -> np.ndarray:
    """polar.hpp:87-106 for one radius and a vector of angles (linear radii)."""
    nr, na = g.shape
    if r > r_max:
        return np.zeros(theta.shape)
    if r <= 1e-9:
        return np.full(theta.shape, g[0].mean())
    u = min(max(r / r_max * nr - 0.5, 0.0), float(nr - 1))
    j0 = min(int(u), nr - 1)
    j1 = min(j0 + 1, nr - 1)
    tu = u - j0
    v = theta / (2 * math.pi) * na
    v = v - np.floor(v / na) * na
    m0 = v.astype(np.int64) % na
    m1 = (m0 + 1) % na
    tv = v - np.floor(v)
    return ((1 - tu) * ((1 - tv) * g[j0, m0] + tv * g[j0, m1]) +
            tu * ((1 - tv) * g[j1, m0] + tv * g[j1, m1]))


def refine_rotation(query: np.ndarray, target: np.ndarray, r_max: float,
                    n_steps: int = 360) -> float:
    """contour.hpp:119-138: the angle phi on a uniform grid minimising
    sum |target(j, m) - query(r_j, theta_m - phi)|^2 (first minimum)."""
    nr, na = query.shape
    theta = 2 * math.pi * np.arange(na) / na
    radii = (np.arange(nr) + 0.5) * r_max / nr
    best, best_err = 0.0, np.inf
    for s in range(n_steps):
        phi = 2 * math.pi * s / n_steps
        err = 0.0
        for j in range(nr):
            q = _polar_sample(query, r_max, radii[j], theta - phi)
            err += float(np.sum((target[j] - q) ** 2))
        if err < best_err:
            best_err, best = err, phi
    return float(normalize_angle(best))


def match_contours(query: ContourScene, target: ContourScene, qx: float, qy: float, eps: float,
                   K: int, top_n: int = 9) -> list:
    """contour.hpp:143-189.  The scatter over the target (xconv_fast) runs on the GPU."""
    frame = normalize_angle(query.normal_angle + math.pi)  # opposite orientation
    try:
        vf = build_vote_filter(query.signal, frame, qx, qy, eps)
    except ValueError:
        raise ValueError("empty contour region") from None
    R = vf.radius
    n_radii = max(4, 2 * R)
    n_angles = max(32, 8 * ((R + 3) // 4) * 4)
    # a per-call filter build: decomposed on the GPU (freq_filter.hpp:63-89)
    F = decompose_rotation2(vf.weights, float(R), float(R), int(K), n_radii, n_angles, R + 0.5,
                            device=True)
    resp = xconv_fast(target.signal, XformField.rotation(target.normal_angle), F)
    real = np.ascontiguousarray(resp.output.real, np.float64)
    peaks = find_peaks(real, eps / 2, 0.1)
    nr_ref, na_ref = max(8, R), 64
    qpatch = resample_polar(query.signal, qx, qy, nr_ref, na_ref, eps)
    out = []
    for p in peaks:
        if len(out) >= top_n:
            break
        tpatch = resample_polar(target.signal, float(p.x), float(p.y), nr_ref, na_ref, eps)
        out.append(ContourMatch(p.x, p.y, refine_rotation(qpatch, tpatch, eps), p.value))
    return out
