"""ctypes binding of the C ABI (include/xconv_b200.h) in lib/libxconv_b200.so.

The product path has no fallback: if the library is missing or no CUDA device
is reachable, calls raise instead of computing anything on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
# XCB_LIB_OVERRIDE: another build of the same library (tools/ab_build.py A/B timing)
LIB_PATH = os.environ.get("XCB_LIB_OVERRIDE") or os.path.join(_PKG, "lib", "libxconv_b200.so")

XC_OK, XC_EINVAL = 0, 2
XC_ROTATION2, XC_SCALE2, XC_ROTATION3 = 0, 1, 2
XC_CORRELATION, XC_CONVOLUTION = 0, 1
XC_F32, XC_F64, XC_C64, XC_C128 = 0, 1, 2, 3
XC_ROW_MAJOR, XC_COL_MAJOR = 0, 1
XC_HOST, XC_DEVICE = 0, 1
XC_FLAG_PERIODIC, XC_FLAG_NO_INNER_DC, XC_FLAG_ACCUMULATE, XC_FLAG_ASYNC = 1, 2, 4, 8
XC_SHARD_BANDS, XC_SHARD_BATCH = 0, 1


class ImageDesc(C.Structure):
    _fields_ = [("height", C.c_int), ("width", C.c_int), ("batch", C.c_int),
                ("signal_dtype", C.c_int), ("param_dtype", C.c_int), ("out_dtype", C.c_int),
                ("layout", C.c_int), ("memory", C.c_int), ("param_per_image", C.c_int),
                ("xform_kind", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("standard_ops", C.c_longlong), ("clamped_pixels", C.c_int),
                ("pad_h", C.c_int), ("pad_w", C.c_int),
                ("seconds_render", C.c_double), ("seconds_fft", C.c_double),
                ("seconds_combine", C.c_double), ("seconds_premultiply", C.c_double),
                ("seconds_h2d", C.c_double), ("seconds_d2h", C.c_double),
                ("seconds_total", C.c_double), ("gpu_launches", C.c_int), ("bands_run", C.c_int),
                ("band_mode", C.c_int)]


EXPORTS = [
    "xc_abi_version", "xc_context_create", "xc_context_destroy", "xc_last_error",
    "xc_context_set_stream", "xc_context_trim", "xc_filter_create", "xc_filter_destroy",
    "xc_filter_num_components", "xc_decompose_rotation2", "xc_decompose_scale2",
    "xc_render_component", "xc_reconstruct", "xc_inner_dc_value", "xc_run", "xc_smooth",
    "xc_anglemax", "xc_find_peaks", "xc_profile_enable", "xc_profile_reset", "xc_profile_get",
    "xc_build_vote_filter", "xc_build_optimal_filter", "xc_detect_pattern",
    "xc_find_peaks_device", "xc_filter3_create", "xc_filter3_destroy", "xc_decompose_rotation3",
    "xc_render_sph_component", "xc_reconstruct3", "xc_sph_harm", "xc_wigner_d", "xc_run3",
    "xc_white_noise", "xc_nccl_unique_id", "xc_context_create_multi", "xc_context_create_rank",
    "xc_context_set_sharding", "xc_context_devices", "xc_context_synchronize",
    "xc_decompose_rotation2_device", "xc_decompose_scale2_device", "xc_debug_check_guards",
    "xc_debug_guard_bytes", "xc_fft2", "xc_debug_pick_pad", "xc_debug_tile_count",
]

_lib = None
_lock = threading.Lock()


class NativeMissing(RuntimeError):
    pass


def lib():
    """Load the CUDA library (raises NativeMissing if it was never built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_2006_13188_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, ip, dp, i, d = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_int, C.c_double
        L.xc_abi_version.restype = i
        L.xc_context_create.argtypes = [i, C.POINTER(vp)]
        L.xc_context_destroy.argtypes = [vp]
        L.xc_context_destroy.restype = None
        L.xc_last_error.argtypes = [vp]
        L.xc_last_error.restype = C.c_char_p
        L.xc_context_set_stream.argtypes = [vp, vp]
        L.xc_context_trim.argtypes = [vp]
        L.xc_filter_create.argtypes = [vp, i, i, ip, i, dp, i, i, d, d, d, C.POINTER(vp)]
        L.xc_filter_destroy.argtypes = [vp]
        L.xc_filter_destroy.restype = None
        L.xc_filter_num_components.argtypes = [vp]
        L.xc_decompose_rotation2.argtypes = [dp, i, i, i, d, d, i, i, i, d, ip, dp, ip]
        L.xc_decompose_scale2.argtypes = [dp, i, i, i, d, d, i, i, i, d, d, d, ip, dp, ip]
        try:  # (absent from older builds timed by tools/ab_kernels.py)
            L.xc_fft2.argtypes = [vp, i, i, i, i, i, vp, vp]
            L.xc_debug_check_guards.argtypes = [vp, ip, C.c_char_p, i]
            L.xc_debug_guard_bytes.argtypes = []
            L.xc_debug_pick_pad.argtypes = [i]
            L.xc_debug_tile_count.argtypes = [i, i]
            L.xc_decompose_rotation2_device.argtypes = [vp, dp, i, i, i, d, d, i, i, i, d, ip,
                                                        dp, ip]
            L.xc_decompose_scale2_device.argtypes = [vp, dp, i, i, i, d, d, i, i, i, d, d, d,
                                                     ip, dp, ip]
        except AttributeError:
            if not os.environ.get("XCB_LIB_OVERRIDE"):
                raise
        L.xc_render_component.argtypes = [vp, i, i, i, d, d, i, dp]
        L.xc_reconstruct.argtypes = [vp, i, i, d, d, ip, i, i, dp]
        L.xc_inner_dc_value.argtypes = [vp, dp]
        L.xc_run.argtypes = [vp, vp, i, C.POINTER(ImageDesc), vp, vp, ip, i, C.c_uint, vp,
                             C.POINTER(Stats)]
        L.xc_smooth.argtypes = [vp, vp, C.POINTER(ImageDesc), vp, vp, i, vp, C.POINTER(Stats)]
        L.xc_anglemax.argtypes = [vp, vp, C.POINTER(ImageDesc), vp, ip, i, i, vp, ip,
                                  C.POINTER(Stats)]
        L.xc_find_peaks.argtypes = [vp, i, i, i, i, d, d, ip, ip, dp, i, ip]
        L.xc_build_vote_filter.argtypes = [dp, dp, i, i, i, d, d, d, i, dp, ip]
        L.xc_build_optimal_filter.argtypes = [dp, i, i, i, d, d, d, i, dp, ip]
        L.xc_detect_pattern.argtypes = [vp, C.POINTER(ImageDesc), vp, dp, i, d, i, i, i, vp, ip,
                                        ip, dp, i, ip, C.POINTER(Stats)]
        L.xc_find_peaks_device.argtypes = [vp, vp, i, i, i, i, d, d, ip, ip, dp, i, ip]
        L.xc_filter3_create.argtypes = [i, i, d, dp, C.POINTER(vp)]
        L.xc_filter3_destroy.argtypes = [vp]
        L.xc_filter3_destroy.restype = None
        L.xc_decompose_rotation3.argtypes = [dp, i, i, i, d, d, d, i, i, d, i, i, dp]
        L.xc_render_sph_component.argtypes = [vp, i, i, i, i, i, i, d, d, d, dp]
        L.xc_reconstruct3.argtypes = [vp, i, i, i, d, d, d, ip, i, dp]
        L.xc_sph_harm.argtypes = [i, i, d, d, dp]
        L.xc_wigner_d.argtypes = [i, dp, dp]
        L.xc_white_noise.argtypes = [C.c_ulonglong, i, i, i, dp]
        L.xc_run3.argtypes = [vp, vp, i, i, i, i, vp, i, vp, ip, i, i, vp, C.POINTER(Stats)]
        L.xc_nccl_unique_id.argtypes = [vp]
        L.xc_context_create_multi.argtypes = [i, ip, C.POINTER(vp)]
        L.xc_context_create_rank.argtypes = [i, vp, i, i, C.POINTER(vp)]
        L.xc_context_set_sharding.argtypes = [vp, i]
        L.xc_context_devices.argtypes = [vp, ip, ip]
        L.xc_context_synchronize.argtypes = [vp]
        L.xc_profile_enable.argtypes = [vp, i]
        L.xc_profile_reset.argtypes = [vp]
        L.xc_profile_get.argtypes = [vp, i, C.c_char_p, i, dp, C.POINTER(C.c_longlong)]
        _lib = L
        return L


def check(rc: int, ctx=None):
    if rc == XC_OK:
        return
    msg = lib().xc_last_error(ctx).decode()
    if rc == XC_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise RuntimeError(f"xconv_b200 error {rc}: {msg}")


def _nccl_first():
    """Map torch's NCCL before the library loads one: a process that later
    imports torch needs torch's (newer) libnccl.so.2, and the loader keeps the
    first libnccl.so.2 it maps."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for Context.rank()."""
    _nccl_first()
    buf = C.create_string_buffer(128)
    check(lib().xc_nccl_unique_id(buf), None)
    return buf.raw


class Context:
    """One xc_context: a single device, or (Context.multi / Context.rank) a
    group whose xc_run / xc_smooth shard the bands across GPUs and reduce
    with NCCL inside the library."""

    def __init__(self, device: int = 0, _handle=None):
        if _handle is None:
            L = lib()
            h = C.c_void_p()
            check(L.xc_context_create(int(device), C.byref(h)), None)
            _handle = h
        self.handle = _handle
        self.device = device

    @classmethod
    def multi(cls, devices, shard: int = XC_SHARD_BANDS) -> "Context":
        """One process driving several devices (a device listed twice reduces
        with peer copies instead of NCCL)."""
        _nccl_first()
        ids = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        check(lib().xc_context_create_multi(len(devices), ids, C.byref(h)), None)
        c = cls(int(devices[0]), _handle=h)
        if shard != XC_SHARD_BANDS:
            check(lib().xc_context_set_sharding(h, int(shard)), h)
        return c

    @classmethod
    def rank(cls, device: int, nccl_id: bytes, rank: int, nranks: int) -> "Context":
        """One process per GPU: every rank calls with the same arguments, rank 0
        receives the band-summed result."""
        _nccl_first()
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        h = C.c_void_p()
        check(lib().xc_context_create_rank(int(device), buf, int(rank), int(nranks), C.byref(h)),
              None)
        return cls(int(device), _handle=h)

    def synchronize(self):
        check(lib().xc_context_synchronize(self.handle), self.handle)

    def devices(self):
        """(number of devices or ranks, whether the reduce is NCCL)."""
        n, u = C.c_int(), C.c_int()
        check(lib().xc_context_devices(self.handle, C.byref(n), C.byref(u)), self.handle)
        return n.value, bool(u.value)

    def set_stream(self, stream_ptr: int | None):
        check(lib().xc_context_set_stream(self.handle, C.c_void_p(stream_ptr or 0)), self.handle)

    def profile(self, enable: bool | None = None, reset: bool = False) -> dict:
        """Per-stage device time {stage: (total_ms, launches)}."""
        L = lib()
        if enable is not None:
            check(L.xc_profile_enable(self.handle, int(enable)), self.handle)
        out = {}
        cnt = L.xc_profile_get(self.handle, -1, None, 0, None, None)
        for i in range(max(cnt, 0)):
            name = C.create_string_buffer(64)
            ms = C.c_double()
            n = C.c_longlong()
            L.xc_profile_get(self.handle, i, name, 64, C.byref(ms), C.byref(n))
            out[name.value.decode()] = (ms.value, n.value)
        if reset:
            check(L.xc_profile_reset(self.handle), self.handle)
        return out

    def check_guards(self):
        """(guard zones changed, first buffer name) -- XCB_GUARD debug mode."""
        n = C.c_int(0)
        name = C.create_string_buffer(128)
        check(lib().xc_debug_check_guards(self.handle, C.byref(n), name, 128), self.handle)
        return n.value, name.value.decode()

    def trim(self):
        check(lib().xc_context_trim(self.handle), self.handle)

    def __del__(self):
        try:
            if self.handle:
                lib().xc_context_destroy(self.handle)
        except Exception:
            pass


_ctx_local = threading.local()


def context(device: int = 0) -> Context:
    """Per-thread, per-device default context."""
    d = getattr(_ctx_local, "ctx", None)
    if d is None:
        d = _ctx_local.ctx = {}
    if device not in d:
        d[device] = Context(device)
    return d[device]
