"""TEST INFRASTRUCTURE ONLY -- ctypes view of the REFERENCE implementation.

oracle/_ref/libxconv_ref.so is the reference's own code
(/root/reference/proj/include/xconv/*.hpp, compiled unchanged against the
Eigen-subset shim in oracle/ref_shim by `make -C oracle ref`, wrapped by
oracle/ref_capi.cpp).  Tests use it to pin the CPU restatement
(oracle/xconv_oracle.cpp, oracle.py) and the GPU product to the reference's
actual outputs.  The product package never imports this module.

Grids are numpy arrays indexed [y, x]; filters are oracle.Filter /
FreqFilter2-like objects (group, K, ks, comps (n_rows, nc), n_radii, n_angles,
r_max, r_min, r_domain).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
_LIB_PATH = os.path.join(REF_DIR, "libxconv_ref.so")
REF_SOURCES = "/root/reference/proj"
REF_TESTS = ["test_fft", "test_field", "test_polar", "test_decompose", "test_sph", "test_wigner",
             "test_engine2d", "test_engine_scale", "test_engine3d", "test_smooth", "test_detect",
             "test_ecd", "test_contour", "test_lic", "test_io"]
_lib = None


def build() -> str | None:
    """Compile the reference (make -C oracle ref) where its sources exist; on
    the GPU box (no /root/reference) the prebuilt oracle/_ref is used."""
    if os.path.isdir(REF_SOURCES):
        subprocess.run(["make", "-s", "-j8", "-C", _HERE, "ref"], check=True,
                       capture_output=True)
    return _LIB_PATH if os.path.exists(_LIB_PATH) else None


def available() -> bool:
    return os.path.exists(_LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{_LIB_PATH} missing: run `make -C oracle ref` where "
                               "/root/reference exists")
        L = C.CDLL(_LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _c128(a):
    return np.ascontiguousarray(np.asarray(a, np.complex128))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, np.float64))


def _check(rc):
    if rc == 2:
        raise ValueError(lib().ref_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


def _fargs(F):
    ks = np.ascontiguousarray(np.asarray(F.ks, np.int32))
    comps = np.asfortranarray(np.asarray(F.comps, np.complex128))  # column-major (n_rows, nc)
    keep = (ks, comps)
    return keep, [int(F.group), int(F.K), _ip(ks), len(ks),
                  comps.ctypes.data_as(C.POINTER(C.c_double)), int(F.n_radii), int(F.n_angles),
                  C.c_double(F.r_max), C.c_double(F.r_min), C.c_double(F.r_domain)]


class Filter:
    def __init__(self, group, K, ks, comps, n_radii, n_angles, r_max, r_min=0.0, r_domain=0.0):
        self.group, self.K = int(group), int(K)
        self.ks = np.asarray(ks, np.int32)
        self.comps = np.asarray(comps, np.complex128)
        self.n_radii, self.n_angles = int(n_radii), int(n_angles)
        self.r_max, self.r_min, self.r_domain = float(r_max), float(r_min), float(r_domain)

    def n_components(self) -> int:
        return len(self.ks)

    def index_of(self, k: int) -> int:
        return int(np.nonzero(self.ks == k)[0][0])


def next_fast_size(n: int) -> int:
    return lib().ref_next_fast_size(int(n))


def fft2(a, inverse=False):
    """fft.hpp:20-53 (the reference's own fft2)."""
    x = _c128(a)
    out = np.zeros(x.shape, np.complex128)
    _check(lib().ref_fft2(_dp(x.view(np.float64)), x.shape[0], x.shape[1], int(bool(inverse)),
                          _dp(out.view(np.float64))))
    return out


def filter2_fft(sig, filt, fcx, fcy, correlate, periodic=False):
    s, f = _c128(sig), _c128(filt)
    out = np.zeros(s.shape, np.complex128)
    _check(lib().ref_filter2_fft(_dp(s.view(np.float64)), s.shape[0], s.shape[1],
                                 _dp(f.view(np.float64)), f.shape[0], f.shape[1], int(fcx),
                                 int(fcy), int(bool(correlate)), int(bool(periodic)),
                                 _dp(out.view(np.float64))))
    return out


def _decomp(fn, filt, *args, n_rows, K):
    f = _c128(filt)
    nk = 2 * (K // 2) + 1
    ks = np.zeros(nk, np.int32)
    comps = np.zeros(n_rows * nk, np.complex128)
    nc = C.c_int(0)
    _check(fn(_dp(f.view(np.float64)), f.shape[0], f.shape[1], *args, _ip(ks),
              _dp(comps.view(np.float64)), C.byref(nc)))
    return ks[:nc.value], comps[:n_rows * nc.value].reshape(nc.value, n_rows).T.copy()


def decompose_rotation2(filt, cx, cy, K, n_radii, n_angles, r_max) -> Filter:
    """freq_filter.hpp:63-89 (the reference's own code)."""
    ks, comps = _decomp(lib().ref_decompose_rotation2, filt, C.c_double(cx), C.c_double(cy),
                        int(K), int(n_radii), int(n_angles), C.c_double(r_max),
                        n_rows=int(n_radii), K=int(K))
    return Filter(0, K, ks, comps, n_radii, n_angles, r_max)


def decompose_scale2(filt, cx, cy, K, n_radii, n_angles, r_min, r_max, r_domain=0.0) -> Filter:
    """freq_filter.hpp:92-129 (the reference's own code)."""
    ks, comps = _decomp(lib().ref_decompose_scale2, filt, C.c_double(cx), C.c_double(cy),
                        int(K), int(n_radii), int(n_angles), C.c_double(r_min),
                        C.c_double(r_max), C.c_double(r_domain), n_rows=int(n_angles), K=int(K))
    D = r_domain if r_domain > 0 else r_max
    return Filter(1, K, ks, comps, n_radii, n_angles, r_max, r_min, D)


def render_component(F, ci, width, height, cx, cy):
    keep, fa = _fargs(F)
    out = np.zeros((height, width), np.complex128)
    _check(lib().ref_render_component(*fa, int(ci), int(width), int(height), C.c_double(cx),
                                      C.c_double(cy), _dp(out.view(np.float64))))
    return out


def xfast(mode, H, kind, param, F, components=None, periodic=False, nthreads=1):
    """xcorr_fast (mode 0) / xconv_fast (mode 1) of the reference.  Returns
    (output complex [h, w], standard_ops)."""
    Hc, P = _c128(H), _f64(param)
    keep, fa = _fargs(F)
    comp = np.ascontiguousarray(np.asarray(components or [], np.int32))
    out = np.zeros(Hc.shape, np.complex128)
    ops = C.c_longlong(0)
    _check(lib().ref_xfast(int(mode), _dp(Hc.view(np.float64)), Hc.shape[0], Hc.shape[1],
                           int(kind), _dp(P), *fa, _ip(comp) if len(comp) else None, len(comp),
                           int(bool(periodic)), int(nthreads), _dp(out.view(np.float64)),
                           C.byref(ops)))
    return out, ops.value


def xcorr_fast(H, kind, param, F, components=None, periodic=False, nthreads=1):
    return xfast(0, H, kind, param, F, components, periodic, nthreads)


def xconv_fast(H, kind, param, F, components=None, periodic=False, nthreads=1):
    return xfast(1, H, kind, param, F, components, periodic, nthreads)


def smooth_adaptive(H, kind, param, F, normalize_signal=True):
    """engine.hpp:385-419 of the reference: (output real, standard_ops, clamped)."""
    Hr, P = _f64(np.real(H)), _f64(param)
    keep, fa = _fargs(F)
    out = np.zeros(Hr.shape)
    ops, cl = C.c_longlong(0), C.c_int(0)
    _check(lib().ref_smooth_adaptive(_dp(Hr), Hr.shape[0], Hr.shape[1], int(kind), _dp(P), *fa,
                                     int(bool(normalize_signal)), _dp(out), C.byref(ops),
                                     C.byref(cl)))
    return out, ops.value, cl.value


def find_peaks(resp, radius, threshold_frac=0.5, max_out=1 << 16):
    r = _f64(resp)
    xs, ys = np.zeros(max_out, np.int32), np.zeros(max_out, np.int32)
    vals = np.zeros(max_out)
    n = lib().ref_find_peaks(_dp(r), r.shape[0], r.shape[1], C.c_double(radius),
                             C.c_double(threshold_frac), _ip(xs), _ip(ys), _dp(vals), max_out)
    return [(int(xs[i]), int(ys[i]), float(vals[i])) for i in range(min(n, max_out))]


def detect_pattern(pattern, px, py, eps, image, K, max_out=4096):
    """build_optimal_filter + detect_pattern of the reference: (response, peaks, ops)."""
    P, I = _f64(pattern), _f64(image)
    resp = np.zeros(I.shape)
    xs, ys = np.zeros(max_out, np.int32), np.zeros(max_out, np.int32)
    vals = np.zeros(max_out)
    n, ops = C.c_int(0), C.c_longlong(0)
    _check(lib().ref_detect_pattern(_dp(P), P.shape[0], P.shape[1], C.c_double(px),
                                    C.c_double(py), C.c_double(eps), _dp(I), I.shape[0],
                                    I.shape[1], int(K), _dp(resp), _ip(xs), _ip(ys), _dp(vals),
                                    max_out, C.byref(n), C.byref(ops)))
    pk = [(int(xs[i]), int(ys[i]), float(vals[i])) for i in range(min(n.value, max_out))]
    return resp, pk, ops.value
