"""Host-side mirror of the reference 3D rotation API.

Same names, argument meaning and error behaviour as the reference
(proj/include/xconv/sph.hpp, wigner.hpp, engine3d.hpp):

    decompose_rotation3 -> SphFilter3              (sph.hpp:161-188, host)
    render_sph_component / reconstruct3 / sph_harm (sph.hpp:37-47, 194-221, host)
    wigner_d(l, q) -> (2l+1)^2 block               (wigner.hpp:64-88, host)
    xcorr_fast_3d(H, T, F, plan) -> Response3      (engine3d.hpp:270-302, GPU)
    xconv_fast_3d(H, T, F, plan) -> Response3      (engine3d.hpp:306-335, GPU)

Volumes are numpy arrays indexed [z, y, x] (Field3 is x fastest,
field.hpp:67-85).  A rotation3 XformField holds quaternions (w, x, y, z) as a
(nz, ny, nx, 4) array (XformField::rotation3d, field.hpp:160-175).  The
filtering runs on the GPU through xc_run3 (k_3d.cu); there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .engine import XConvPlan, XformField, XformKind, XMode


def rotation3d(quats) -> XformField:
    """XformField::rotation3d (field.hpp:160-175): (nz, ny, nx, 4) quaternions
    (w, x, y, z); non-unit ones are renormalized (|norm - 1| > 1e-12)."""
    q = np.array(quats, dtype=np.float64)
    if q.ndim != 4 or q.shape[-1] != 4:
        raise ValueError("quaternion count does not match grid dims")
    nr = np.linalg.norm(q, axis=-1, keepdims=True)
    q = np.where(np.abs(nr - 1.0) > 1e-12, q / nr, q)
    return XformField(XformKind.rotation3, q)


class SphFilter3:
    """Per-shell spherical harmonic coefficients (sph.hpp:130-157): coeffs is
    (n_radii, (K+1)^2) complex, column l(l+1)+m."""

    def __init__(self, K, n_radii, r_max, coeffs):
        self.K = int(K)
        self.n_radii = int(n_radii)
        self.r_max = float(r_max)
        self.coeffs = np.asarray(coeffs, dtype=np.complex128).copy()
        self._h = None

    def coeff(self, shell, l, m) -> complex:
        return complex(self.coeffs[shell, l * (l + 1) + m])

    def handle(self):
        if self._h is None:
            cm = np.asfortranarray(self.coeffs)  # Eigen column-major
            out = C.c_void_p()
            N.check(N.lib().xc_filter3_create(self.K, self.n_radii, self.r_max,
                                              cm.ctypes.data_as(C.POINTER(C.c_double)),
                                              C.byref(out)))
            self._h = out
        return self._h

    def __del__(self):
        try:
            if self._h is not None:
                N.lib().xc_filter3_destroy(self._h)
        except Exception:
            pass


@dataclass
class Response3:  # engine.hpp Response3 (engine3d.hpp:283-299)
    output: np.ndarray
    plan: XConvPlan
    standard_ops: int = 0
    seconds: dict = field(default_factory=dict)
    gpu_launches: int = 0


def _vol(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def decompose_rotation3(volume, cx, cy, cz, K, n_radii, r_max, n_theta=0,
                        n_phi=0) -> SphFilter3:
    """sph.hpp:161-188 (host, once per filter)."""
    v = _vol(volume)
    nz, ny, nx = v.shape
    out = np.zeros((int(n_radii), (int(K) + 1) ** 2), np.complex128, order="F")
    N.check(N.lib().xc_decompose_rotation3(v.ctypes.data_as(C.POINTER(C.c_double)), nx, ny, nz,
                                           float(cx), float(cy), float(cz), int(K), int(n_radii),
                                           float(r_max), int(n_theta), int(n_phi),
                                           out.ctypes.data_as(C.POINTER(C.c_double))))
    return SphFilter3(K, n_radii, r_max, out)


def render_sph_component(F: SphFilter3, l, m_radial, m_angular, nx, ny, nz, cx, cy, cz):
    """sph.hpp:194-212."""
    out = np.zeros((nz, ny, nx), np.complex128)
    N.check(N.lib().xc_render_sph_component(F.handle(), int(l), int(m_radial), int(m_angular),
                                            nx, ny, nz, float(cx), float(cy), float(cz),
                                            out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def reconstruct3(F: SphFilter3, nx, ny, nz, cx, cy, cz, degrees=None):
    """sph.hpp:215-221."""
    out = np.zeros((nz, ny, nx), np.complex128)
    d = None if degrees is None else np.ascontiguousarray(np.asarray(degrees, np.int32))
    N.check(N.lib().xc_reconstruct3(F.handle(), nx, ny, nz, float(cx), float(cy), float(cz),
                                    None if d is None else d.ctypes.data_as(C.POINTER(C.c_int)),
                                    -1 if d is None else len(d),
                                    out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def sph_harm(l, m, theta, phi) -> complex:
    """sph.hpp:37-47."""
    o = np.zeros(2)
    N.check(N.lib().xc_sph_harm(int(l), int(m), float(theta), float(phi),
                                o.ctypes.data_as(C.POINTER(C.c_double))))
    return complex(o[0], o[1])


def wigner_d(l, q) -> np.ndarray:
    """wigner.hpp:64-88: D[m_to + l, m_from + l]."""
    qa = np.ascontiguousarray(np.asarray(q, dtype=np.float64))
    out = np.zeros((2 * max(int(l), 0) + 1,) * 2, np.complex128)
    N.check(N.lib().xc_wigner_d(int(l), qa.ctypes.data_as(C.POINTER(C.c_double)),
                                out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


_DT = {np.dtype(np.float32): N.XC_F32, np.dtype(np.float64): N.XC_F64,
       np.dtype(np.complex64): N.XC_C64, np.dtype(np.complex128): N.XC_C128}


def _fast3(mode, H, T: XformField, F: SphFilter3, plan: XConvPlan | None,
           device: int = 0) -> Response3:
    plan = XConvPlan() if plan is None else XConvPlan(plan.mode, plan.group,
                                                      list(plan.components), plan.periodic)
    if T.kind != XformKind.rotation3:  # engine3d.hpp:273
        raise ValueError("needs a rotation3 field")
    sig = np.asarray(getattr(H, "values", H))
    if sig.dtype not in _DT:
        sig = sig.astype(np.complex128 if np.iscomplexobj(sig) else np.float64)
    sig = np.ascontiguousarray(sig)
    q = np.ascontiguousarray(np.asarray(T.values, dtype=np.float64))
    if sig.ndim != 3 or q.shape != sig.shape + (4,):
        raise ValueError("signal and transformation field dims differ")
    nz, ny, nx = sig.shape
    out = np.zeros(sig.shape, np.complex128)
    deg = np.ascontiguousarray(np.asarray(plan.components, np.int32))
    ctx = N.context(device)
    st = N.Stats()
    N.check(N.lib().xc_run3(ctx.handle, F.handle(), int(mode), nx, ny, nz, sig.ctypes.data,
                            _DT[sig.dtype], q.ctypes.data,
                            deg.ctypes.data_as(C.POINTER(C.c_int)) if len(deg) else None,
                            len(deg), N.XC_HOST, out.ctypes.data, C.byref(st)), ctx.handle)
    plan.mode = XMode(mode)
    plan.group = XformKind.rotation3
    return Response3(out, plan, int(st.standard_ops),
                     {"fft": st.seconds_fft, "total": st.seconds_total}, int(st.gpu_launches))


def xcorr_fast_3d(H, T: XformField, F: SphFilter3, plan: XConvPlan | None = None) -> Response3:
    """engine3d.hpp:270-302: out = sum_{l,m,m'} conj(D^l_{m'm}(R_p)) (H * V_{l m m'})(p)."""
    return _fast3(XMode.correlation, H, T, F, plan)


def xconv_fast_3d(H, T: XformField, F: SphFilter3, plan: XConvPlan | None = None) -> Response3:
    """engine3d.hpp:306-335: out = sum_{l,m,m'} (H D^l_{m'm}) conv V_{l m m'}."""
    return _fast3(XMode.convolution, H, T, F, plan)


def steer_filter3(F: SphFilter3, q) -> SphFilter3:
    """Rotate a 3D filter by mixing each degree's coefficients per radial shell
    with D^l(q) (xconv_cli.cpp:191-204, the steer3d subcommand)."""
    out = F.coeffs.copy()
    for l in range(F.K + 1):
        D = wigner_d(l, q)
        cols = slice(l * l, (l + 1) * (l + 1))  # l(l+1)+m for m = -l..l
        out[:, cols] = F.coeffs[:, cols] @ D.T
    return SphFilter3(F.K, F.n_radii, F.r_max, out)
