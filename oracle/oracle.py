"""TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU oracle (xconv_oracle.cpp).

The oracle is a double-precision restatement of the reference 2D path
(/root/reference/proj/include/xconv/*.hpp, see the citations in
xconv_oracle.cpp).  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs import this module; the product package never does.

Grids are numpy arrays indexed [y, x] (the reference's values(y, x)).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc/g++ only)."""
    # make is a no-op when the library is newer than its sources; on a box
    # without the sources' build tools the prebuilt library is used as is
    try:
        subprocess.run(["make", "-s", "-C", _HERE] + (["-B"] if force else []), check=True,
                       capture_output=True)
    except (OSError, subprocess.CalledProcessError):
        if not os.path.exists(_LIB_PATH):
            raise
    return _LIB_PATH


class _OrFilter(C.Structure):
    _fields_ = [
        ("group", C.c_int), ("K", C.c_int), ("nc", C.c_int),
        ("ks", C.POINTER(C.c_int)), ("comps", C.POINTER(C.c_double)),
        ("n_radii", C.c_int), ("n_angles", C.c_int),
        ("r_max", C.c_double), ("r_min", C.c_double), ("r_domain", C.c_double),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        L.or_rng_new.restype = C.c_void_p
        L.or_rng_new.argtypes = [C.c_uint64]
        L.or_rng_free.argtypes = [C.c_void_p]
        L.or_rng_next.restype = C.c_uint64
        L.or_rng_next.argtypes = [C.c_void_p]
        L.or_rng_uniform.restype = C.c_double
        L.or_rng_uniform.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.or_wigner_small_d.restype = C.c_double
        for name in ("or_random_field", "or_random_smooth_filter", "or_annular_filter",
                     "or_random_rotation_field", "or_random_scale_field", "or_random_field3",
                     "or_random_smooth_filter3", "or_random_quaternion",
                     "or_random_rotation3_field", "or_euler_zyz", "or_sphere_grid"):
            getattr(L, name).restype = None
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _check(rc: int):
    if rc == 2:
        raise ValueError(lib().or_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib().or_last_error().decode())


@dataclass
class Filter:
    """FreqFilter2 (freq_filter.hpp:21-46); comps is (n_rows, nc) complex."""
    group: int
    K: int
    ks: np.ndarray
    comps: np.ndarray
    n_radii: int
    n_angles: int
    r_max: float
    r_min: float = 0.0
    r_domain: float = 0.0
    _keep: list = field(default_factory=list, repr=False)

    def n_components(self) -> int:
        return len(self.ks)

    def index_of(self, k: int) -> int:
        return int(np.nonzero(np.asarray(self.ks) == k)[0][0])

    def domain_top(self) -> float:
        return self.r_domain if self.r_domain > 0 else self.r_max

    def omega(self) -> float:
        return 2.0 * np.pi / np.log(self.domain_top() / self.r_min)


def _cfilter(F) -> _OrFilter:
    ks = np.ascontiguousarray(np.asarray(F.ks, dtype=np.int32))
    comps = _c128(F.comps)
    s = _OrFilter(int(F.group), int(F.K), len(ks), _ip(ks), _dp(comps.view(np.float64)),
                  int(F.n_radii), int(F.n_angles), float(F.r_max), float(F.r_min),
                  float(F.r_domain))
    s._keep = (ks, comps)  # keep buffers alive
    return s


# ----------------------------------------------------------------- FFT layer

def next_fast_size(n: int) -> int:
    return lib().or_next_fast_size(int(n))


def fft2(a, inverse=False) -> np.ndarray:
    a = _c128(a).copy()
    lib().or_fft2(_dp(a.view(np.float64)), a.shape[0], a.shape[1], int(inverse))
    return a


def filter2_fft(sig, filt, fcx, fcy, correlate, periodic=False) -> np.ndarray:
    sig, filt = _c128(sig), _c128(filt)
    out = np.zeros_like(sig)
    lib().or_filter2_fft(_dp(sig.view(np.float64)), sig.shape[0], sig.shape[1],
                         _dp(filt.view(np.float64)), filt.shape[0], filt.shape[1],
                         int(fcx), int(fcy), int(correlate), int(periodic),
                         _dp(out.view(np.float64)))
    return out


def correlate_direct(H, F, fcx, fcy) -> np.ndarray:
    H, F = _c128(H), _c128(F)
    out = np.zeros_like(H)
    lib().or_correlate_direct(_dp(H.view(np.float64)), H.shape[0], H.shape[1],
                              _dp(F.view(np.float64)), F.shape[0], F.shape[1], fcx, fcy,
                              _dp(out.view(np.float64)))
    return out


def convolve_direct(H, F, fcx, fcy) -> np.ndarray:
    H, F = _c128(H), _c128(F)
    out = np.zeros_like(H)
    lib().or_convolve_direct(_dp(H.view(np.float64)), H.shape[0], H.shape[1],
                             _dp(F.view(np.float64)), F.shape[0], F.shape[1], fcx, fcy,
                             _dp(out.view(np.float64)))
    return out


# ----------------------------------------------------------- decomposition

def decompose_rotation2(filt, cx, cy, K, n_radii, n_angles, r_max) -> Filter:
    filt = _c128(filt)
    nc_max = 2 * (K // 2) + 1
    ks = np.zeros(nc_max, np.int32)
    comps = np.zeros((max(n_radii, 1), nc_max), np.complex128)
    nc = C.c_int(0)
    _check(lib().or_decompose_rotation2(
        _dp(filt.view(np.float64)), filt.shape[1], filt.shape[0], C.c_double(cx),
        C.c_double(cy), int(K), int(n_radii), int(n_angles), C.c_double(r_max), _ip(ks),
        _dp(comps.view(np.float64)), C.byref(nc)))
    return Filter(0, K, ks[: nc.value].copy(), comps[:, : nc.value].copy(), n_radii,
                  n_angles, float(r_max))


def decompose_scale2(filt, cx, cy, K, n_radii, n_angles, r_min, r_max,
                     r_domain=0.0) -> Filter:
    filt = _c128(filt)
    nc_max = 2 * (K // 2) + 1
    ks = np.zeros(nc_max, np.int32)
    comps = np.zeros((max(n_angles, 1), nc_max), np.complex128)
    nc = C.c_int(0)
    _check(lib().or_decompose_scale2(
        _dp(filt.view(np.float64)), filt.shape[1], filt.shape[0], C.c_double(cx),
        C.c_double(cy), int(K), int(n_radii), int(n_angles), C.c_double(r_min),
        C.c_double(r_max), C.c_double(r_domain), _ip(ks), _dp(comps.view(np.float64)),
        C.byref(nc)))
    D = r_domain if r_domain > 0 else r_max
    return Filter(1, K, ks[: nc.value].copy(), comps[:, : nc.value].copy(), n_radii,
                  n_angles, float(r_max), float(r_min), float(D))


def component_value(F, ci, r, theta) -> complex:
    out = np.zeros(2)
    lib().or_component_value(C.byref(_cfilter(F)), int(ci), C.c_double(r),
                             C.c_double(theta), _dp(out))
    return complex(out[0], out[1])


def render_component(F, ci, width, height, cx, cy) -> np.ndarray:
    out = np.zeros((height, width), np.complex128)
    lib().or_render_component(C.byref(_cfilter(F)), int(ci), int(width), int(height),
                              C.c_double(cx), C.c_double(cy), _dp(out.view(np.float64)))
    return out


def inner_dc_value(F) -> complex:
    out = np.zeros(2)
    lib().or_inner_dc_value(C.byref(_cfilter(F)), _dp(out))
    return complex(out[0], out[1])


def reconstruct(F, width, height, cx, cy, subset=None) -> np.ndarray:
    out = np.zeros((height, width), np.complex128)
    sub = None if subset is None else np.ascontiguousarray(np.asarray(subset, np.int32))
    lib().or_reconstruct(C.byref(_cfilter(F)), int(width), int(height), C.c_double(cx),
                         C.c_double(cy), None if sub is None else _ip(sub),
                         -1 if sub is None else len(sub), _dp(out.view(np.float64)))
    return out


def synthesize_polar(F, subset=None) -> np.ndarray:
    out = np.zeros((F.n_radii, F.n_angles), np.complex128)
    sub = None if subset is None else np.ascontiguousarray(np.asarray(subset, np.int32))
    lib().or_synthesize_polar(C.byref(_cfilter(F)), None if sub is None else _ip(sub),
                              -1 if sub is None else len(sub), _dp(out.view(np.float64)))
    return out


# ------------------------------------------------------------------ engine

def _xfast(mode, H, kind, param, F, components, periodic, nthreads):
    H = _c128(H)
    param = _f64(param)
    assert param.shape == H.shape
    out = np.zeros_like(H)
    ops = C.c_longlong(0)
    secs = np.zeros(4)
    comp = None if not components else np.ascontiguousarray(np.asarray(components, np.int32))
    _check(lib().or_xfast(int(mode), _dp(H.view(np.float64)), H.shape[0], H.shape[1],
                          int(kind), _dp(param), C.byref(_cfilter(F)),
                          None if comp is None else _ip(comp),
                          0 if comp is None else len(comp), int(periodic),
                          _dp(out.view(np.float64)), C.byref(ops), _dp(secs),
                          int(nthreads)))
    return out, ops.value, dict(zip(("render", "fft", "combine", "premultiply"), secs))


def xcorr_fast(H, kind, param, F, components=None, periodic=False, nthreads=1):
    """engine.hpp:286-326. Returns (output, standard_ops, seconds)."""
    return _xfast(0, H, kind, param, F, components, periodic, nthreads)


def xconv_fast(H, kind, param, F, components=None, periodic=False, nthreads=1):
    """engine.hpp:331-373. Returns (output, standard_ops, seconds)."""
    return _xfast(1, H, kind, param, F, components, periodic, nthreads)


def smooth_adaptive(H, kind, param, F, normalize_signal=True, nthreads=1):
    """engine.hpp:385-419. Returns (output_real, standard_ops, clamped_pixels)."""
    H = _c128(H)
    param = _f64(param)
    out = np.zeros(H.shape, np.float64)
    ops = C.c_longlong(0)
    cl = C.c_int(0)
    _check(lib().or_smooth_adaptive(_dp(H.view(np.float64)), H.shape[0], H.shape[1],
                                    int(kind), _dp(param), C.byref(_cfilter(F)),
                                    int(normalize_signal), _dp(out), C.byref(ops),
                                    C.byref(cl), int(nthreads)))
    return out, ops.value, cl.value


def _brute(mode, H, kind, param, F, eps, table_radii, table_angles):
    H = _c128(H)
    param = _f64(param)
    out = np.zeros_like(H)
    _check(lib().or_xbrute(int(mode), _dp(H.view(np.float64)), H.shape[0], H.shape[1],
                           int(kind), _dp(param), C.byref(_cfilter(F)), C.c_double(eps),
                           int(table_radii), int(table_angles), _dp(out.view(np.float64))))
    return out


def xcorr_brute(H, kind, param, F, eps=0.0, table_radii=0, table_angles=0):
    return _brute(0, H, kind, param, F, eps, table_radii, table_angles)


def xconv_brute(H, kind, param, F, eps=0.0, table_radii=0, table_angles=0):
    return _brute(1, H, kind, param, F, eps, table_radii, table_angles)


def spectral_oracle(mode, H, kind, param, F):
    H = _c128(H)
    param = _f64(param)
    out = np.zeros_like(H)
    _check(lib().or_spectral_oracle(int(mode), _dp(H.view(np.float64)), H.shape[0],
                                    H.shape[1], int(kind), _dp(param), C.byref(_cfilter(F)),
                                    _dp(out.view(np.float64))))
    return out


def spectral_oracle_at(mode, H, kind, param, F, pys, pxs):
    """Spectral oracle at sampled pixels (float32 real H / param)."""
    H = np.ascontiguousarray(np.asarray(H, np.float32))
    param = np.ascontiguousarray(np.asarray(param, np.float32))
    pys = np.ascontiguousarray(np.asarray(pys, np.int32))
    pxs = np.ascontiguousarray(np.asarray(pxs, np.int32))
    out = np.zeros(len(pys), np.complex128)
    fp = C.POINTER(C.c_float)
    _check(lib().or_spectral_oracle_at(int(mode), H.ctypes.data_as(fp), H.shape[0], H.shape[1],
                                       int(kind), param.ctypes.data_as(fp), C.byref(_cfilter(F)),
                                       _ip(pys), _ip(pxs), len(pys), _dp(out.view(np.float64))))
    return out


def find_peaks(resp, radius, threshold_frac=0.5, max_out=1 << 16):
    resp = _f64(resp)
    xs = np.zeros(max_out, np.int32)
    ys = np.zeros(max_out, np.int32)
    vals = np.zeros(max_out)
    n = lib().or_find_peaks(_dp(resp), resp.shape[0], resp.shape[1], C.c_double(radius),
                            C.c_double(threshold_frac), _ip(xs), _ip(ys), _dp(vals), max_out)
    n = min(n, max_out)
    return [(int(xs[i]), int(ys[i]), float(vals[i])) for i in range(n)]


def gaussian_blur(img, sigma) -> np.ndarray:
    img = _f64(img)
    out = np.zeros_like(img)
    lib().or_gaussian_blur(_dp(img), img.shape[0], img.shape[1], C.c_double(sigma), _dp(out))
    return out


def gradient(img):
    img = _f64(img)
    mag = np.zeros_like(img)
    d = np.zeros_like(img)
    lib().or_gradient(_dp(img), img.shape[0], img.shape[1], _dp(mag), _dp(d))
    return mag, d


def build_vote_filter(weight, frame, px, py, eps, nearest=False):
    """vote_filter.hpp:62-81 -> (weights (2R+1, 2R+1), R)."""
    weight = _f64(weight)
    frame = _f64(frame)
    R = int(np.ceil(eps))
    out = np.zeros((2 * R + 1, 2 * R + 1))
    r = C.c_int(0)
    _check(lib().or_build_vote_filter(_dp(weight), _dp(frame), weight.shape[0], weight.shape[1],
                                      C.c_double(px), C.c_double(py), C.c_double(eps),
                                      int(nearest), _dp(out), C.byref(r)))
    return out, r.value


def build_optimal_filter(pattern, px, py, eps, nearest=False):
    """vote_filter.hpp:83-91 -> (weights (2R+1, 2R+1), R)."""
    pattern = _f64(pattern)
    R = int(np.ceil(eps))
    out = np.zeros((2 * R + 1, 2 * R + 1))
    r = C.c_int(0)
    _check(lib().or_build_optimal_filter(_dp(pattern), pattern.shape[0], pattern.shape[1],
                                         C.c_double(px), C.c_double(py), C.c_double(eps),
                                         int(nearest), _dp(out), C.byref(r)))
    return out, r.value


def detect_pattern(image, weights, radius, eps, K, n_radii=0, n_angles=0, max_peaks=4096):
    """vote_filter.hpp:146-168 -> (response, [(x, y, value)], standard_ops)."""
    image = _f64(image)
    weights = _f64(weights)
    h, w = image.shape
    resp = np.zeros((h, w))
    xs = np.zeros(max_peaks, np.int32)
    ys = np.zeros(max_peaks, np.int32)
    vs = np.zeros(max_peaks)
    n = C.c_int(0)
    ops = C.c_longlong(0)
    _check(lib().or_detect_pattern(_dp(image), h, w, _dp(weights), int(radius), C.c_double(eps),
                                   int(K), int(n_radii), int(n_angles), _dp(resp), _ip(xs),
                                   _ip(ys), _dp(vs), max_peaks, C.byref(n), C.byref(ops)))
    k = min(n.value, max_peaks)
    return resp, [(int(xs[i]), int(ys[i]), float(vs[i])) for i in range(k)], ops.value


def anglemax(G, ks, n_angles=360):
    """G: (nc, h, w) complex band responses.  Returns (score, argmax)."""
    G = _c128(G)
    ks = np.ascontiguousarray(np.asarray(ks, np.int32))
    nc, h, w = G.shape
    score = np.zeros((h, w))
    arg = np.zeros((h, w), np.int32)
    lib().or_anglemax(_dp(G.view(np.float64)), _ip(ks), nc, h, w, int(n_angles),
                      _dp(score), _ip(arg))
    return score, arg


def band_responses(H, F, ks=None, nthreads=1) -> np.ndarray:
    """(nk, h, w) complex G_k = H (*) F_k (correlation, no steering)."""
    H = _c128(H)
    h, w = H.shape
    ks = np.ascontiguousarray(np.asarray(F.ks if ks is None else ks, np.int32))
    G = np.zeros((len(ks), h, w), np.complex128)
    cf = _cfilter(F)
    _check(lib().or_band_responses(_dp(H.view(np.float64)), h, w, C.byref(cf), _ip(ks),
                                   len(ks), int(nthreads), _dp(G.view(np.float64))))
    return G


def anglemax_mt(G, ks, n_angles=360, nthreads=1):
    """anglemax() with rows split across threads (same max / first-argmax)."""
    G = _c128(G)
    ks = np.ascontiguousarray(np.asarray(ks, np.int32))
    nc, h, w = G.shape
    score = np.zeros((h, w))
    arg = np.zeros((h, w), np.int32)
    lib().or_anglemax_mt(_dp(G.view(np.float64)), _ip(ks), nc, h, w, int(n_angles),
                         int(nthreads), _dp(score), _ip(arg))
    return score, arg


def direct_at(mode, H, kind, param, F, pys, pxs, nthreads=1) -> np.ndarray:
    """xcorr_fast (mode 0) / xconv_fast (mode 1) at pixels (pys, pxs) by direct
    summation over the rendered bands (no FFT)."""
    H = _c128(H)
    h, w = H.shape
    pys = np.ascontiguousarray(np.asarray(pys, np.int32))
    pxs = np.ascontiguousarray(np.asarray(pxs, np.int32))
    out = np.zeros(len(pys), np.complex128)
    cf = _cfilter(F)
    _check(lib().or_direct_at(int(mode), _dp(H.view(np.float64)), h, w, int(kind),
                              _dp(_f64(param)), C.byref(cf), _ip(pys), _ip(pxs), len(pys),
                              int(nthreads), _dp(out.view(np.float64))))
    return out


# ------------------------------------------------------------------ fixtures

class Rng:
    """std::mt19937_64 shared across fixtures, as in proj/tests/helpers.hpp."""

    def __init__(self, seed: int):
        self._h = C.c_void_p(lib().or_rng_new(int(seed)))

    def __del__(self):
        try:
            lib().or_rng_free(self._h)
        except Exception:
            pass

    def next(self) -> int:
        return lib().or_rng_next(self._h)

    def uniform(self, a, b) -> float:
        return lib().or_rng_uniform(self._h, a, b)

    def random_field(self, w, h, complex_valued=False) -> np.ndarray:
        out = np.zeros((h, w), np.complex128)
        lib().or_random_field(self._h, int(w), int(h), int(complex_valued),
                              _dp(out.view(np.float64)))
        return out

    def random_smooth_filter(self, radius, n_bumps=6, envelope_frac=0.35) -> np.ndarray:
        S = 2 * radius + 1
        out = np.zeros((S, S), np.complex128)
        lib().or_random_smooth_filter(self._h, int(radius), int(n_bumps),
                                      C.c_double(envelope_frac), _dp(out.view(np.float64)))
        return out

    def annular_filter(self, R, r0_frac=0.55, sr_frac=0.18) -> np.ndarray:
        S = 2 * R + 1
        out = np.zeros((S, S), np.complex128)
        lib().or_annular_filter(self._h, int(R), C.c_double(r0_frac), C.c_double(sr_frac),
                                _dp(out.view(np.float64)))
        return out

    def random_rotation_field(self, w, h) -> np.ndarray:
        out = np.zeros((h, w))
        lib().or_random_rotation_field(self._h, int(w), int(h), _dp(out))
        return out

    def random_scale_field(self, w, h, lo=0.5, hi=2.0) -> np.ndarray:
        out = np.zeros((h, w))
        lib().or_random_scale_field(self._h, int(w), int(h), C.c_double(lo), C.c_double(hi),
                                    _dp(out))
        return out


def white_noise(width, height, seed) -> np.ndarray:
    """lic.hpp:9-17: std::mt19937_64(seed); f.at(x, y) = (rng() >> 11) * 2^-53
    in y-major order.  [height][width]."""
    h = C.c_void_p(lib().or_rng_new(int(seed) & (2**64 - 1)))
    try:
        out = np.zeros((int(height), int(width)))
        for y in range(int(height)):
            for x in range(int(width)):
                out[y, x] = float(lib().or_rng_next(h) >> 11) * 2.0 ** -53
    finally:
        lib().or_rng_free(h)
    return out


def anisotropic_gaussian(length, width) -> np.ndarray:
    """lic.hpp:20-32 (loop form)."""
    R = int(np.ceil(2.5 * length))
    f = np.zeros((2 * R + 1, 2 * R + 1))
    for y in range(-R, R + 1):
        for x in range(-R, R + 1):
            if float(x * x + y * y) > float(R) * R:
                continue
            f[y + R, x + R] = np.exp(-float(x) * x / (2 * length * length)
                                     - float(y) * y / (2 * width * width))
    return f


def lic(angles, length, width, seed, normalized=True, K=16, nthreads=1) -> np.ndarray:
    """lic.hpp:37-55 over the restated decomposition and engine (rotation2)."""
    if not (length > width) or not (width > 0):
        raise ValueError("need length > width > 0")
    angles = _f64(angles)
    h, w = angles.shape
    noise = white_noise(w, h, seed)
    kern = anisotropic_gaussian(length, width)
    R = (kern.shape[1] - 1) // 2
    F = decompose_rotation2(kern, float(R), float(R), int(K), max(8, R), max(64, 4 * int(K)),
                            R + 0.5)
    if normalized:
        return smooth_adaptive(noise, 0, angles, F, True, nthreads)[0]
    return xconv_fast(noise, 0, angles, F, nthreads=nthreads)[0].real


def structure_tensor(img, sigma=2.0):
    """proj/tests/helpers.hpp:161-191: (orientation, coherence) of the
    gradient structure tensor blurred by sigma; orientation is the streak
    direction (perpendicular to the dominant gradient), normalized to [-pi, pi)."""
    mag, d = gradient(img)
    gx, gy = mag * np.cos(d), mag * np.sin(d)
    jxx = gaussian_blur(gx * gx, sigma)
    jxy = gaussian_blur(gx * gy, sigma)
    jyy = gaussian_blur(gy * gy, sigma)
    tr = jxx + jyy
    det = np.sqrt(np.maximum(0.0, (jxx - jyy) ** 2 + 4 * jxy * jxy))
    o = 0.5 * np.arctan2(2 * jxy, jxx - jyy) + np.pi / 2
    o = np.fmod(o + np.pi, 2 * np.pi)
    o = np.where(o < 0, o + 2 * np.pi, o) - np.pi
    coh = np.where(tr > 1e-12, det / np.where(tr > 1e-12, tr, 1.0), 0.0)
    return o, coh


def orientation_distance(a, b):
    """proj/tests/helpers.hpp:194-198 (undirected, mod pi)."""
    d = np.fmod(np.abs(a - b), np.pi)
    return np.minimum(d, np.pi - d)


def rel_l2(a, b) -> float:
    """helpers.hpp:10-14"""
    a = np.asarray(a)
    b = np.asarray(b)
    n = np.sqrt(np.sum(np.abs(a - b) ** 2))
    d = np.sqrt(np.sum(np.abs(b) ** 2))
    return float(n / d) if d > 0 else float(n)


# ------------------------------------------------------------------ 3D
# Volumes are numpy arrays indexed [z, y, x] (Field3, x fastest, field.hpp:67-85);
# quaternion fields are (nz, ny, nx, 4) arrays of (w, x, y, z).

@dataclass
class Filter3:
    """SphFilter3 (sph.hpp:130-157): coeffs (n_radii, (K+1)^2) complex, column l(l+1)+m."""
    K: int
    n_radii: int
    r_max: float
    coeffs: np.ndarray

    def coeff(self, shell, l, m) -> complex:
        return complex(self.coeffs[shell, l * (l + 1) + m])


def _f3(F: Filter3):
    return int(F.K), int(F.n_radii), C.c_double(F.r_max), _dp(_c128(F.coeffs).view(np.float64))


def decompose_rotation3(vol, cx, cy, cz, K, n_radii, r_max, n_theta=0, n_phi=0) -> Filter3:
    """sph.hpp:161-188"""
    v = _c128(vol)
    nz, ny, nx = v.shape
    out = np.zeros((n_radii, (K + 1) ** 2), np.complex128)
    _check(lib().or_decompose_rotation3(_dp(v.view(np.float64)), nx, ny, nz, C.c_double(cx),
                                        C.c_double(cy), C.c_double(cz), int(K), int(n_radii),
                                        C.c_double(r_max), int(n_theta), int(n_phi),
                                        _dp(out.view(np.float64))))
    return Filter3(int(K), int(n_radii), float(r_max), out)


def render_sph_component(F: Filter3, l, m_radial, m_angular, nx, ny, nz, cx, cy, cz):
    """sph.hpp:194-212"""
    out = np.zeros((nz, ny, nx), np.complex128)
    keep = _c128(F.coeffs)
    _check(lib().or_render_sph_component(int(F.K), int(F.n_radii), C.c_double(F.r_max),
                                         _dp(keep.view(np.float64)), int(l), int(m_radial),
                                         int(m_angular), nx, ny, nz, C.c_double(cx),
                                         C.c_double(cy), C.c_double(cz),
                                         _dp(out.view(np.float64))))
    return out


def reconstruct3(F: Filter3, nx, ny, nz, cx, cy, cz, degrees=None):
    """sph.hpp:215-221"""
    out = np.zeros((nz, ny, nx), np.complex128)
    keep = _c128(F.coeffs)
    d = np.ascontiguousarray(np.asarray(degrees if degrees is not None else [], np.int32))
    _check(lib().or_reconstruct3(int(F.K), int(F.n_radii), C.c_double(F.r_max),
                                 _dp(keep.view(np.float64)), nx, ny, nz, C.c_double(cx),
                                 C.c_double(cy), C.c_double(cz), _ip(d),
                                 -1 if degrees is None else len(d), _dp(out.view(np.float64))))
    return out


def sph_harm(l, m, theta, phi) -> complex:
    """sph.hpp:37-47"""
    o = np.zeros(2)
    _check(lib().or_sph_harm(int(l), int(m), C.c_double(theta), C.c_double(phi), _dp(o)))
    return complex(o[0], o[1])


def sphere_grid(n_theta, n_phi):
    """SphereGrid (sph.hpp:52-86): (theta, weight)."""
    th = np.zeros(n_theta)
    w = np.zeros(n_theta)
    lib().or_sphere_grid(int(n_theta), int(n_phi), _dp(th), _dp(w))
    return th, w


def euler_zyz(q):
    """wigner.hpp:40-57"""
    qa = _f64(q)
    o = np.zeros(3)
    lib().or_euler_zyz(_dp(qa), _dp(o))
    return tuple(o)


def wigner_d(l, q) -> np.ndarray:
    """wigner.hpp:64-88: D[m_to + l, m_from + l]"""
    qa = _f64(q)
    o = np.zeros((2 * l + 1, 2 * l + 1), np.complex128) if l >= 0 else np.zeros(1, np.complex128)
    _check(lib().or_wigner_d(int(l), _dp(qa), _dp(o.view(np.float64))))
    return o


def filter3_fft(sig, filt, fcx, fcy, fcz, correlate):
    """fft.hpp:175-207"""
    s = _c128(sig)
    f = _c128(filt)
    out = np.zeros(s.shape, np.complex128)
    _check(lib().or_filter3_fft(_dp(s.view(np.float64)), s.shape[2], s.shape[1], s.shape[0],
                                _dp(f.view(np.float64)), f.shape[2], f.shape[1], f.shape[0],
                                int(fcx), int(fcy), int(fcz), int(bool(correlate)),
                                _dp(out.view(np.float64))))
    return out


def xfast3(mode, H, quats, F: Filter3, degrees=None):
    """engine3d.hpp:267-335 (mode 0 xcorr_fast_3d, 1 xconv_fast_3d): (output, standard_ops)."""
    h = _c128(H)
    q = _f64(quats)
    nz, ny, nx = h.shape
    if q.shape != (nz, ny, nx, 4):
        raise ValueError("signal and transformation field dims differ")
    out = np.zeros(h.shape, np.complex128)
    keep = _c128(F.coeffs)
    d = np.ascontiguousarray(np.asarray(degrees if degrees is not None else [], np.int32))
    ops = C.c_longlong(0)
    _check(lib().or_xfast3(int(mode), _dp(h.view(np.float64)), nx, ny, nz, _dp(q), int(F.K),
                           int(F.n_radii), C.c_double(F.r_max), _dp(keep.view(np.float64)),
                           _ip(d), len(d), _dp(out.view(np.float64)), C.byref(ops)))
    return out, ops.value


def exact3(mode, H, quats, F: Filter3):
    """test_engine3d.cpp:37-67: rotated band-limited reconstruction, spatial loops."""
    h = _c128(H)
    q = _f64(quats)
    nz, ny, nx = h.shape
    out = np.zeros(h.shape, np.complex128)
    keep = _c128(F.coeffs)
    _check(lib().or_exact3(int(mode), _dp(h.view(np.float64)), nx, ny, nz, _dp(q), int(F.K),
                           int(F.n_radii), C.c_double(F.r_max), _dp(keep.view(np.float64)),
                           _dp(out.view(np.float64))))
    return out


def _random_field3(self, nx, ny, nz, complex_valued=False):
    out = np.zeros((nz, ny, nx), np.complex128)
    lib().or_random_field3(self._h, nx, ny, nz, int(complex_valued), _dp(out.view(np.float64)))
    return out


def _random_smooth_filter3(self, radius, n_bumps=6, envelope_frac=0.4):
    S = 2 * radius + 1
    out = np.zeros((S, S, S), np.complex128)
    lib().or_random_smooth_filter3(self._h, int(radius), int(n_bumps), C.c_double(envelope_frac),
                                   _dp(out.view(np.float64)))
    return out


def _random_quaternion(self):
    out = np.zeros(4)
    lib().or_random_quaternion(self._h, _dp(out))
    return out


def _random_rotation3_field(self, nx, ny, nz):
    out = np.zeros((nz, ny, nx, 4))
    lib().or_random_rotation3_field(self._h, nx * ny * nz, _dp(out))
    return out


Rng.random_field3 = _random_field3
Rng.random_smooth_filter3 = _random_smooth_filter3
Rng.random_quaternion = _random_quaternion
Rng.random_rotation3_field = _random_rotation3_field


def quat_mul(a, b):
    """Hamilton product (Eigen Quaternion operator*)."""
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw])


def quat_matrix(q):
    """Eigen Quaternion::toRotationMatrix."""
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
