"""Host-side mirror of the reference operator API for the hot path.

Same names, argument meaning and error behaviour as the reference C++ API
(proj/include/xconv/engine.hpp, freq_filter.hpp, field.hpp, vote_filter.hpp):

    decompose_rotation2 / decompose_scale2 -> FreqFilter2   (freq_filter.hpp:63-129)
    render_component / reconstruct / inner_dc_value          (freq_filter.hpp:165-235)
    xcorr_fast(H, T, F, plan) -> Response2                   (engine.hpp:286-326)
    xconv_fast(H, T, F, plan) -> Response2                   (engine.hpp:331-373)
    smooth_adaptive(H, T, F, normalize_signal) -> SmoothResult (engine.hpp:385-419)
    anglemax(H, F, n_angles)                                 (new)
    find_peaks(resp, radius, threshold_frac)                 (vote_filter.hpp:107-134)

std::invalid_argument surfaces as ValueError with the reference's message.
Every call goes through the C ABI into the sm_100a kernels; nothing here
computes a result on the CPU.  Grids are numpy arrays indexed [y, x] (the
reference's values(y, x)); batches are (B, H, W).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _native as N


class XformKind(IntEnum):  # field.hpp:129
    rotation2 = 0
    scale2 = 1
    rotation3 = 2


class XMode(IntEnum):  # engine.hpp:10
    correlation = 0
    convolution = 1


# ------------------------------------------------------------------ fields

class XformField:
    """Per-pixel transformation parameters (field.hpp:133-185).

    Angles are kept as given (the steering phase e^{ik theta} is 2 pi periodic,
    so the reference's normalize_angle, field.hpp:122-127, is implicit);
    `angle` returns the normalized copy on demand."""

    def __init__(self, kind: XformKind, values: np.ndarray):
        self.kind = XformKind(kind)
        self.values = values

    @staticmethod
    def rotation(angles) -> "XformField":
        return XformField(XformKind.rotation2, np.asarray(angles))

    @staticmethod
    def scaling(scales) -> "XformField":
        s = np.asarray(scales)
        if not (np.all(s > 0) and np.all(np.isfinite(s))):  # field.hpp:151-152
            raise ValueError("scale field must be strictly positive and finite")
        return XformField(XformKind.scale2, s)

    @property
    def angle(self) -> np.ndarray:
        a = np.fmod(self.values.astype(np.float64) + math.pi, 2 * math.pi)
        a = np.where(a < 0, a + 2 * math.pi, a)
        return a - math.pi

    @property
    def scale(self) -> np.ndarray:
        return self.values

    @property
    def log_scale(self) -> np.ndarray:
        return np.log(self.values)

    def width(self) -> int:
        return int(self.values.shape[-1])

    def height(self) -> int:
        return int(self.values.shape[-2])


# ----------------------------------------------------------------- filters

class FreqFilter2:
    """Steerable band decomposition of a 2D filter (freq_filter.hpp:21-46).

    comps is (n_rows, nc) complex: n_rows = n_radii for rotation2 (radial
    profiles), n_angles for scale2 (angular profiles)."""

    def __init__(self, group, K, ks, comps, n_radii, n_angles, r_max, r_min=0.0,
                 r_domain=0.0):
        self.group = XformKind(group)
        self.K = int(K)
        self.ks = np.asarray(ks, dtype=np.int32).copy()
        self.comps = np.asarray(comps, dtype=np.complex128).copy()
        self.n_radii = int(n_radii)
        self.n_angles = int(n_angles)
        self.r_max = float(r_max)
        self.r_min = float(r_min)
        self.r_domain = float(r_domain)
        self._handles = {}

    # freq_filter.hpp:33-45
    def n_components(self) -> int:
        return len(self.ks)

    def index_of(self, k: int) -> int:
        hits = np.nonzero(self.ks == k)[0]
        if len(hits) == 0:
            raise ValueError("frequency not retained")
        return int(hits[0])

    def domain_top(self) -> float:
        return self.r_domain if self.r_domain > 0 else self.r_max

    def log_period(self) -> float:
        return math.log(self.domain_top() / self.r_min)

    def omega(self) -> float:
        return 2.0 * math.pi / self.log_period()

    def hermitian(self) -> bool:
        """F_{-k} = conj(F_k) for every retained band (a real filter): the test the
        library applies before its Hermitian half-band mode (host_filter.cpp)."""
        tol = 1e-12 * max(float(np.abs(self.comps).max(initial=0.0)), 1e-300)
        for ci, k in enumerate(self.ks):
            hits = np.nonzero(self.ks == -k)[0]
            if len(hits) == 0:
                return False
            if np.abs(self.comps[:, hits[-1]] - np.conj(self.comps[:, ci])).max(initial=0.0) > tol:
                return False
        return True

    def handle(self, ctx: N.Context | None = None):
        """The xc_filter handle (host object; device spectra are cached in it)."""
        h = self._handles.get(0)
        if h is None:
            cm = np.asfortranarray(self.comps)  # Eigen column-major
            ks = np.ascontiguousarray(self.ks)
            out = C.c_void_p()
            N.check(N.lib().xc_filter_create(
                None, int(self.group), self.K, ks.ctypes.data_as(C.POINTER(C.c_int)),
                len(ks), cm.ctypes.data_as(C.POINTER(C.c_double)), self.n_radii,
                self.n_angles, self.r_max, self.r_min, self.r_domain, C.byref(out)))
            h = self._handles[0] = out
        return h

    def __del__(self):
        try:
            for h in self._handles.values():
                N.lib().xc_filter_destroy(h)
        except Exception:
            pass


def _filter_image(filt) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(filt, dtype=np.complex128))


def _decompose_ctx(device):
    """device=False/None: the host decomposition; True: this thread's default
    context; an int: that device's context; a Context: itself."""
    if device is None or device is False:
        return None
    if device is True:
        return N.context(0)
    return device if isinstance(device, N.Context) else N.context(int(device))


def decompose_rotation2(filt, cx, cy, K, n_radii, n_angles, r_max, device=None) -> FreqFilter2:
    """freq_filter.hpp:63-89.  Host by default (once per filter); device=True
    (or a device id / Context) runs the polar resampling and the band DFT on
    the GPU (xc_decompose_rotation2_device), for per-call filter builds."""
    f = _filter_image(filt)
    nc = 2 * (int(K) // 2) + 1
    ks = np.zeros(nc, np.int32)
    comps = np.zeros((max(int(n_radii), 1), nc), np.complex128, order="F")
    got = C.c_int(0)
    args = (f.ctypes.data_as(C.POINTER(C.c_double)), f.shape[0], f.shape[1], N.XC_ROW_MAJOR,
            float(cx), float(cy), int(K), int(n_radii), int(n_angles), float(r_max),
            ks.ctypes.data_as(C.POINTER(C.c_int)), comps.ctypes.data_as(C.POINTER(C.c_double)),
            C.byref(got))
    ctx = _decompose_ctx(device)
    if ctx is None:
        N.check(N.lib().xc_decompose_rotation2(*args))
    else:
        N.check(N.lib().xc_decompose_rotation2_device(ctx.handle, *args), ctx.handle)
    return FreqFilter2(XformKind.rotation2, K, ks, comps, n_radii, n_angles, r_max)


def decompose_scale2(filt, cx, cy, K, n_radii, n_angles, r_min, r_max,
                     r_domain=0.0, device=None) -> FreqFilter2:
    """freq_filter.hpp:91-129 (host by default; device= as decompose_rotation2)."""
    f = _filter_image(filt)
    nc = 2 * (int(K) // 2) + 1
    ks = np.zeros(nc, np.int32)
    comps = np.zeros((max(int(n_angles), 1), nc), np.complex128, order="F")
    got = C.c_int(0)
    args = (f.ctypes.data_as(C.POINTER(C.c_double)), f.shape[0], f.shape[1], N.XC_ROW_MAJOR,
            float(cx), float(cy), int(K), int(n_radii), int(n_angles), float(r_min), float(r_max),
            float(r_domain), ks.ctypes.data_as(C.POINTER(C.c_int)),
            comps.ctypes.data_as(C.POINTER(C.c_double)), C.byref(got))
    ctx = _decompose_ctx(device)
    if ctx is None:
        N.check(N.lib().xc_decompose_scale2(*args))
    else:
        N.check(N.lib().xc_decompose_scale2_device(ctx.handle, *args), ctx.handle)
    D = r_domain if r_domain > 0 else r_max
    return FreqFilter2(XformKind.scale2, K, ks, comps, n_radii, n_angles, r_max, r_min, D)


def fft2(a, inverse: bool = False, device=0) -> np.ndarray:
    """fft.hpp:20-53 on the GPU with the pipeline's own transforms
    (xc_fft2): forward unscaled, inverse scaled 1/n; complex64 in gives
    complex64 out, anything else complex128 (computed in fp32)."""
    x = np.asarray(a)
    x = np.ascontiguousarray(x if x.dtype in (np.complex64, np.complex128)
                             else x.astype(np.complex128))
    if x.ndim != 2:
        raise ValueError("fft2 takes a 2D grid")
    out = np.zeros_like(x)
    ctx = _context(device)
    N.check(N.lib().xc_fft2(ctx.handle, x.shape[0], x.shape[1],
                            N.XC_C64 if x.dtype == np.complex64 else N.XC_C128, N.XC_HOST,
                            int(bool(inverse)), x.ctypes.data, out.ctypes.data), ctx.handle)
    return out


def render_component(F: FreqFilter2, ci, width, height, cx, cy) -> np.ndarray:
    """freq_filter.hpp:172-184."""
    out = np.zeros((height, width), np.complex128)
    N.check(N.lib().xc_render_component(F.handle(), int(ci), int(width), int(height),
                                        float(cx), float(cy), N.XC_ROW_MAJOR,
                                        out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def reconstruct(F: FreqFilter2, width, height, cx, cy, subset=None) -> np.ndarray:
    """freq_filter.hpp:216-235."""
    out = np.zeros((height, width), np.complex128)
    sub = None if subset is None else np.ascontiguousarray(np.asarray(subset, np.int32))
    N.check(N.lib().xc_reconstruct(F.handle(), int(width), int(height), float(cx),
                                   float(cy),
                                   None if sub is None else sub.ctypes.data_as(C.POINTER(C.c_int)),
                                   -1 if sub is None else len(sub), N.XC_ROW_MAJOR,
                                   out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def inner_dc_value(F: FreqFilter2) -> complex:
    """freq_filter.hpp:165-169."""
    v = np.zeros(2)
    N.check(N.lib().xc_inner_dc_value(F.handle(), v.ctypes.data_as(C.POINTER(C.c_double))))
    return complex(v[0], v[1])


# ------------------------------------------------------------------ engine

@dataclass
class XConvPlan:  # engine.hpp:16-21
    mode: XMode = XMode.correlation
    group: XformKind = XformKind.rotation2
    components: list = field(default_factory=list)
    periodic: bool = False


@dataclass
class Response2:  # engine.hpp:23-29
    output: np.ndarray
    plan: XConvPlan
    standard_ops: int = 0
    seconds: dict = field(default_factory=dict)
    gpu_launches: int = 0


@dataclass
class SmoothResult:  # engine.hpp:377-382
    output: np.ndarray
    standard_ops: int = 0
    clamped_pixels: int = 0


_SIG_DT = {np.dtype(np.float32): N.XC_F32, np.dtype(np.float64): N.XC_F64,
           np.dtype(np.complex64): N.XC_C64, np.dtype(np.complex128): N.XC_C128}


def _signal(H):
    a = np.asarray(getattr(H, "values", H))
    if a.dtype not in _SIG_DT:
        a = a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)
    return np.ascontiguousarray(a)


def _param(T: XformField, shape):
    p = np.asarray(T.values)
    if p.dtype not in (np.float32, np.float64):
        p = p.astype(np.float64)
    if p.shape[-2:] != shape[-2:]:
        raise ValueError("signal and transformation field dims differ")
    return np.ascontiguousarray(p)


def _desc(sig, par, out_dt, kind, memory=N.XC_HOST):
    b = 1 if sig.ndim == 2 else sig.shape[0]
    per = 1 if (par is not None and par.ndim == 3) else 0
    return N.ImageDesc(sig.shape[-2], sig.shape[-1], b, _SIG_DT[sig.dtype],
                       N.XC_F64 if par is None or par.dtype == np.float64 else N.XC_F32,
                       out_dt, N.XC_ROW_MAJOR, memory, per, int(kind))


def _seconds(st: N.Stats) -> dict:
    return {"render": st.seconds_render, "fft": st.seconds_fft, "combine": st.seconds_combine,
            "premultiply": st.seconds_premultiply, "h2d": st.seconds_h2d,
            "d2h": st.seconds_d2h, "total": st.seconds_total}


def _context(device) -> N.Context:
    """`device` is a device ordinal (the thread's default context on it) or an
    explicit N.Context (e.g. N.Context.multi([0, 1, ...]) for band sharding)."""
    return device if isinstance(device, N.Context) else N.context(int(device))


def _fast(mode: XMode, H, T: XformField, F: FreqFilter2, plan: XConvPlan | None,
          device=0, inner_dc: bool = True) -> Response2:
    plan = XConvPlan() if plan is None else XConvPlan(plan.mode, plan.group,
                                                      list(plan.components), plan.periodic)
    sig = _signal(H)
    par = _param(T, sig.shape)
    wide = sig.dtype in (np.float64, np.complex128)
    out = np.zeros(sig.shape, np.complex128 if wide else np.complex64)
    ctx = _context(device)
    d = _desc(sig, par, N.XC_C128 if wide else N.XC_C64, T.kind)
    comp = np.ascontiguousarray(np.asarray(plan.components, np.int32))
    st = N.Stats()
    flags = N.XC_FLAG_PERIODIC if plan.periodic else 0
    if not inner_dc:  # band-sharded scale runs add the inner-DC term on one rank
        flags |= N.XC_FLAG_NO_INNER_DC
    N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), int(mode), C.byref(d),
                           sig.ctypes.data, par.ctypes.data,
                           comp.ctypes.data_as(C.POINTER(C.c_int)) if len(comp) else None,
                           len(comp), flags, out.ctypes.data, C.byref(st)), ctx.handle)
    plan.mode = mode
    plan.group = T.kind
    return Response2(out, plan, st.standard_ops, _seconds(st), st.gpu_launches)


def xcorr_fast(H, T: XformField, F: FreqFilter2, plan: XConvPlan | None = None,
               ctx=0) -> Response2:
    """Extended correlation (engine.hpp:286-326): out(p) = sum_k e^{i phase_k(p)} (H * F_k)(p).
    ctx: device ordinal or N.Context (a multi-GPU context shards the bands)."""
    return _fast(XMode.correlation, H, T, F, plan, ctx)


def xconv_fast(H, T: XformField, F: FreqFilter2, plan: XConvPlan | None = None,
               ctx=0) -> Response2:
    """Extended convolution (engine.hpp:331-373): sum_k (H e^{-i phase_k}) conv F_k."""
    return _fast(XMode.convolution, H, T, F, plan, ctx)


def smooth_adaptive(H, T: XformField, F: FreqFilter2, normalize_signal: bool = True,
                    device=0) -> SmoothResult:
    """Normalized adaptive smoothing (engine.hpp:385-419)."""
    sig = _signal(H)
    par = _param(T, sig.shape)
    wide = sig.dtype in (np.float64, np.complex128)
    out = np.zeros(sig.shape, np.float64 if wide else np.float32)
    ctx = _context(device)
    d = _desc(sig, par, N.XC_F64 if wide else N.XC_F32, T.kind)
    st = N.Stats()
    N.check(N.lib().xc_smooth(ctx.handle, F.handle(ctx), C.byref(d), sig.ctypes.data,
                              par.ctypes.data, int(bool(normalize_signal)), out.ctypes.data,
                              C.byref(st)), ctx.handle)
    return SmoothResult(out, st.standard_ops, st.clamped_pixels)


def anglemax(H, F: FreqFilter2, n_angles: int = 360, components=None, device: int = 0):
    """Rotation-invariant match score: max over n_angles sampled rotations of
    |sum_k e^{-i k 2 pi s/n} G_k(p)|, G_k = H (*) F_k.
    Returns (score float64/float32, argmax int32)."""
    sig = _signal(H)
    wide = sig.dtype in (np.float64, np.complex128)
    score = np.zeros(sig.shape, np.float64 if wide else np.float32)
    arg = np.zeros(sig.shape, np.int32)
    ctx = N.context(device)
    d = _desc(sig, None, N.XC_F64 if wide else N.XC_F32, XformKind.rotation2)
    comp = np.ascontiguousarray(np.asarray(components or [], np.int32))
    st = N.Stats()
    N.check(N.lib().xc_anglemax(ctx.handle, F.handle(ctx), C.byref(d), sig.ctypes.data,
                                comp.ctypes.data_as(C.POINTER(C.c_int)) if len(comp) else None,
                                len(comp), int(n_angles), score.ctypes.data,
                                arg.ctypes.data_as(C.POINTER(C.c_int)), C.byref(st)),
            ctx.handle)
    return score, arg


@dataclass
class Peak:  # vote_filter.hpp:99-102
    x: int
    y: int
    value: float


def find_peaks(resp, radius: float, threshold_frac: float = 0.5, max_peaks: int = 1 << 16,
               gpu: bool = False, device: int = 0):
    """NMS peaks, sorted by value desc, then y, then x (vote_filter.hpp:107-134).
    gpu=True runs the NMS on the GPU (xc_find_peaks_device; a torch CUDA tensor is
    used in place, a host array is uploaded) -- same peaks as the host version."""
    if gpu:
        return _find_peaks_gpu(resp, radius, threshold_frac, max_peaks, device)
    r = np.ascontiguousarray(np.asarray(resp))
    dt = N.XC_F32 if r.dtype == np.float32 else N.XC_F64
    if dt == N.XC_F64 and r.dtype != np.float64:
        r = r.astype(np.float64)
    xs = np.zeros(max_peaks, np.int32)
    ys = np.zeros(max_peaks, np.int32)
    vs = np.zeros(max_peaks)
    n = C.c_int(0)
    N.check(N.lib().xc_find_peaks(r.ctypes.data, dt, r.shape[0], r.shape[1], N.XC_ROW_MAJOR,
                                  float(radius), float(threshold_frac),
                                  xs.ctypes.data_as(C.POINTER(C.c_int)),
                                  ys.ctypes.data_as(C.POINTER(C.c_int)),
                                  vs.ctypes.data_as(C.POINTER(C.c_double)), max_peaks,
                                  C.byref(n)))
    return [Peak(int(xs[i]), int(ys[i]), float(vs[i])) for i in range(min(n.value, max_peaks))]


def _find_peaks_gpu(resp, radius, threshold_frac, max_peaks, device):
    import torch
    t = resp if isinstance(resp, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(resp))
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    t = t.to(torch.device("cuda", device)).contiguous()
    dt = N.XC_F32 if t.dtype == torch.float32 else N.XC_F64
    xs = np.zeros(max_peaks, np.int32)
    ys = np.zeros(max_peaks, np.int32)
    vs = np.zeros(max_peaks)
    n = C.c_int(0)
    ctx = N.context(device)
    torch.cuda.synchronize(t.device)
    N.check(N.lib().xc_find_peaks_device(ctx.handle, C.c_void_p(t.data_ptr()), dt, t.shape[0],
                                         t.shape[1], N.XC_ROW_MAJOR, float(radius),
                                         float(threshold_frac),
                                         xs.ctypes.data_as(C.POINTER(C.c_int)),
                                         ys.ctypes.data_as(C.POINTER(C.c_int)),
                                         vs.ctypes.data_as(C.POINTER(C.c_double)), max_peaks,
                                         C.byref(n)), ctx.handle)
    return [Peak(int(xs[i]), int(ys[i]), float(vs[i])) for i in range(min(n.value, max_peaks))]


# ---------------------------------------------------------------- detection
# vote_filter.hpp: generalized-Hough pattern detection on the
# hot path -- gradient on the GPU, scatter through xc_run, NMS on the host.

@dataclass
class VoteFilter:  # vote_filter.hpp:8-26
    weights: np.ndarray  # (2R+1, 2R+1) row-major [y][x], non-negative
    radius: int
    eps: float

    def side(self) -> int:
        return 2 * self.radius + 1

    def total_mass(self) -> float:
        return float(self.weights.sum())


@dataclass
class DetectionResult:  # vote_filter.hpp:137-142
    response: np.ndarray
    peaks: list
    standard_ops: int = 0


def _f64_2d(a):
    return np.ascontiguousarray(np.asarray(getattr(a, "values", a), dtype=np.float64))


def build_vote_filter(weight, frame, px: float, py: float, eps: float,
                      nearest: bool = False) -> VoteFilter:
    """Votes of every q with weight(q) > 0 within eps of (px, py), rotated into the
    frame at q (vote_filter.hpp:62-81)."""
    w = _f64_2d(weight)
    f = _f64_2d(frame)
    if f.shape != w.shape:
        raise ValueError("weight and frame dims differ")
    R = int(np.ceil(eps)) if eps > 0 else 0
    out = np.zeros((2 * R + 1, 2 * R + 1))
    r = C.c_int(0)
    N.check(N.lib().xc_build_vote_filter(w.ctypes.data_as(C.POINTER(C.c_double)),
                                         f.ctypes.data_as(C.POINTER(C.c_double)), w.shape[0],
                                         w.shape[1], N.XC_ROW_MAJOR, float(px), float(py),
                                         float(eps), int(nearest),
                                         out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r)))
    return VoteFilter(out, r.value, float(eps))


def build_optimal_filter(pattern, px: float, py: float, eps: float,
                         nearest: bool = False) -> VoteFilter:
    """Optimal filter of a pattern: gradient-magnitude votes in the gradient frame
    (vote_filter.hpp:83-91)."""
    p = _f64_2d(pattern)
    R = int(np.ceil(eps)) if eps > 0 else 0
    out = np.zeros((2 * R + 1, 2 * R + 1))
    r = C.c_int(0)
    N.check(N.lib().xc_build_optimal_filter(p.ctypes.data_as(C.POINTER(C.c_double)), p.shape[0],
                                            p.shape[1], N.XC_ROW_MAJOR, float(px), float(py),
                                            float(eps), int(nearest),
                                            out.ctypes.data_as(C.POINTER(C.c_double)),
                                            C.byref(r)))
    return VoteFilter(out, r.value, float(eps))


def detect_pattern(image, filter: VoteFilter, K: int, n_radii: int = 0, n_angles: int = 0,
                   device: int = 0, max_peaks: int = 1 << 16) -> DetectionResult:
    """Gradient magnitudes vote through the filter's K-band decomposition, steered by
    the gradient directions; peaks by NMS within eps/2 (vote_filter.hpp:146-168)."""
    img = np.ascontiguousarray(np.asarray(getattr(image, "values", image)))
    if np.iscomplexobj(img):
        raise ValueError("gradient requires real field")
    if img.dtype not in (np.float32, np.float64):
        img = img.astype(np.float64)
    wide = img.dtype == np.float64
    h, w = img.shape
    resp = np.zeros((h, w), np.float64 if wide else np.float32)
    d = N.ImageDesc(h, w, 1, N.XC_F64 if wide else N.XC_F32, N.XC_F32,
                    N.XC_F64 if wide else N.XC_F32, N.XC_ROW_MAJOR, N.XC_HOST, 0,
                    XformKind.rotation2)
    wts = np.ascontiguousarray(filter.weights, np.float64)
    xs = np.zeros(max_peaks, np.int32)
    ys = np.zeros(max_peaks, np.int32)
    vs = np.zeros(max_peaks)
    n = C.c_int(0)
    st = N.Stats()
    ctx = N.context(device)
    N.check(N.lib().xc_detect_pattern(ctx.handle, C.byref(d), img.ctypes.data,
                                      wts.ctypes.data_as(C.POINTER(C.c_double)),
                                      int(filter.radius), float(filter.eps), int(K),
                                      int(n_radii), int(n_angles), resp.ctypes.data,
                                      xs.ctypes.data_as(C.POINTER(C.c_int)),
                                      ys.ctypes.data_as(C.POINTER(C.c_int)),
                                      vs.ctypes.data_as(C.POINTER(C.c_double)), max_peaks,
                                      C.byref(n), C.byref(st)), ctx.handle)
    peaks = [Peak(int(xs[i]), int(ys[i]), float(vs[i])) for i in range(min(n.value, max_peaks))]
    return DetectionResult(resp, peaks, int(st.standard_ops))
