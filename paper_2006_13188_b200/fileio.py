"""Wire and disk formats of the reference, host side.

Byte-for-byte the layouts of proj/include/xconv/io.hpp, so files written by
the reference CLI load here and the reverse:

    read_pgm / write_pgm            P5, 8 or 16 bit (big-endian), io.hpp:44-103
    write_pfm_planes / read_pfm_planes
                                    grayscale "Pf" blocks, little-endian fp32,
                                    rows bottom-up, io.hpp:105-162
    write_pfm / read_pfm_field      1 plane real, 2 planes complex, io.hpp:164-183
    write_xform / read_xform        angle / scale planes (4 quaternion planes
                                    for rotation3), io.hpp:185-236
    write_filter / read_filter      XCF1 filter container, io.hpp:238-316

Grids are numpy arrays indexed [y, x] (the reference's values(y, x)).  Errors
are IoError with the reference's message texts.  No GPU work happens here:
these are the callers' formats on either side of the C ABI.
"""
from __future__ import annotations

import struct

import numpy as np

from .engine import FreqFilter2, XformField, XformKind


class IoError(RuntimeError):
    """io.hpp:14-16 (xconv::IoError)."""


# ------------------------------------------------------------------ helpers

_SPACE = b" \t\n\v\f\r"


class _Reader:
    """The subset of std::istream the reference parsers use: `>>` tokens
    (skipping whitespace), get(), peek(), read(n)."""

    def __init__(self, data: bytes):
        self.d = data
        self.i = 0

    def peek(self) -> int:
        return self.d[self.i] if self.i < len(self.d) else -1

    def get(self) -> int:
        c = self.peek()
        if c >= 0:
            self.i += 1
        return c

    def token(self) -> bytes:
        while self.i < len(self.d) and self.d[self.i] in _SPACE:
            self.i += 1
        s = self.i
        while self.i < len(self.d) and self.d[self.i] not in _SPACE:
            self.i += 1
        return self.d[s:self.i]

    def skip_pnm_space(self):  # io.hpp:20-32
        while True:
            c = self.peek()
            if c == ord("#"):
                j = self.d.find(b"\n", self.i)
                self.i = len(self.d) if j < 0 else j + 1
            elif c >= 0 and c in _SPACE:
                self.i += 1
            else:
                return

    def read(self, n: int) -> bytes | None:
        if self.i + n > len(self.d):
            self.i = len(self.d)
            return None
        b = self.d[self.i:self.i + n]
        self.i += n
        return b


def _int_token(r: _Reader, path: str, what: str) -> int:
    t = r.token()
    try:
        return int(t)
    except ValueError:
        raise IoError(f"{path}: {what}") from None


def _slurp(path: str) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError:
        raise IoError("cannot open " + path) from None


def _open_w(path: str):
    try:
        return open(path, "wb")
    except OSError:
        raise IoError("cannot open " + path + " for writing") from None


# ------------------------------------------------------------------ PGM

def read_pgm(path: str) -> np.ndarray:
    """io.hpp:44-81: values / maxval as float64, [y, x]."""
    r = _Reader(_slurp(path))
    if r.token() != b"P5":
        raise IoError(path + ": not a P5 PGM")
    try:
        r.skip_pnm_space()
        w = int(r.token())
        r.skip_pnm_space()
        h = int(r.token())
        r.skip_pnm_space()
        maxval = int(r.token())
    except ValueError:
        raise IoError(path + ": bad PGM header") from None
    r.get()  # single whitespace before the raster
    if w < 1 or h < 1 or maxval < 1 or maxval > 65535:
        raise IoError(path + ": bad PGM header")
    if maxval < 256:
        buf = r.read(w * h)
        if buf is None:
            raise IoError(path + ": truncated PGM raster")
        a = np.frombuffer(buf, np.uint8).astype(np.float64)
    else:
        buf = r.read(w * h * 2)
        if buf is None:
            raise IoError(path + ": truncated PGM raster")
        a = np.frombuffer(buf, ">u2").astype(np.float64)  # big-endian per PNM
    return a.reshape(h, w) / maxval


def write_pgm(path: str, f, maxval: int = 255) -> None:
    """io.hpp:83-103: real part clamped to [0, 1], scaled, rounded half away
    from zero (std::lround)."""
    v = np.real(np.asarray(f)).astype(np.float64)
    if v.ndim != 2:
        raise IoError("PGM needs a 2D field")
    h, w = v.shape
    q = np.floor(np.clip(v, 0.0, 1.0) * maxval + 0.5).astype(np.int64)
    raster = q.astype(np.uint8).tobytes() if maxval < 256 else q.astype(">u2").tobytes()
    with _open_w(path) as out:
        out.write(b"P5\n%d %d\n%d\n" % (w, h, maxval))
        out.write(raster)


# ------------------------------------------------------------------ PFM

def write_pfm_planes(path: str, planes) -> None:
    """io.hpp:112-129: one "Pf" block per plane, fp32 little-endian, rows
    bottom-up."""
    planes = [np.asarray(p, dtype=np.float64) for p in planes]
    if not planes:
        raise IoError("no planes to write")
    with _open_w(path) as out:
        for p in planes:
            h, w = p.shape
            out.write(b"Pf\n%d %d\n-1.0\n" % (w, h))
            out.write(np.ascontiguousarray(p[::-1]).astype("<f4").tobytes())


def read_pfm_planes(path: str) -> list:
    """io.hpp:131-162: every consecutive Pf block (float64 [y, x] grids); the
    scale's sign selects the byte order."""
    r = _Reader(_slurp(path))
    planes = []
    while r.peek() != -1:
        magic = r.token()
        if not magic:
            break
        if magic != b"Pf":
            raise IoError(path + ": expected grayscale Pf plane")
        try:
            w = int(r.token())
            h = int(r.token())
            scale = float(r.token())
        except ValueError:
            raise IoError(path + ": bad PFM header") from None
        r.get()
        if w < 1 or h < 1:
            raise IoError(path + ": bad PFM header")
        buf = r.read(4 * w * h)
        if buf is None:
            raise IoError(path + ": truncated PFM raster")
        a = np.frombuffer(buf, "<f4" if scale < 0 else ">f4").reshape(h, w)
        planes.append(a[::-1].astype(np.float64))
        while r.peek() in (ord("\n"), ord("\r")):
            r.get()
    if not planes:
        raise IoError(path + ": no PFM planes")
    return planes


def _is_real(f) -> bool:  # field.hpp Field2::is_real (imaginary parts exactly 0)
    return not np.iscomplexobj(f) or not np.any(np.imag(f))


def write_pfm(path: str, f) -> None:
    """io.hpp:164-171: a real field is one plane, a complex field two (re, im)."""
    f = np.asarray(f)
    if _is_real(f):
        write_pfm_planes(path, [np.real(f)])
    else:
        write_pfm_planes(path, [np.real(f), np.imag(f)])


def read_pfm_field(path: str) -> np.ndarray:
    """io.hpp:173-183: complex128 [y, x] (imaginary part 0 for one plane)."""
    planes = read_pfm_planes(path)
    if len(planes) not in (1, 2):
        raise IoError(path + ": expected 1 (real) or 2 (complex) planes")
    out = planes[0].astype(np.complex128)
    if len(planes) == 2:
        out = out + 1j * planes[1]
    return out


def write_xform(path: str, T: XformField) -> None:
    """io.hpp:185-210: rotation2 writes the normalized angle plane, scale2 the
    scale plane, rotation3 the (w, x, y, z) planes of a single-slice field."""
    if T.kind == XformKind.rotation2:
        write_pfm_planes(path, [T.angle])
    elif T.kind == XformKind.scale2:
        write_pfm_planes(path, [T.scale])
    else:
        # engine3d.rotation3d layout: (nz, ny, nx, 4) quaternions (w, x, y, z)
        q = np.asarray(T.values)
        if q.ndim != 4 or q.shape[-1] != 4 or q.shape[0] != 1:
            raise IoError("PFM export supports single-slice quaternion fields")
        write_pfm_planes(path, [q[0, ..., i] for i in range(4)])


def read_xform(path: str, kind: XformKind) -> XformField:
    """io.hpp:212-236."""
    planes = read_pfm_planes(path)
    kind = XformKind(kind)
    if kind == XformKind.rotation2:
        if len(planes) != 1:
            raise IoError(path + ": rotation field needs 1 plane")
        return XformField.rotation(planes[0])
    if kind == XformKind.scale2:
        if len(planes) != 1:
            raise IoError(path + ": scale field needs 1 plane")
        return XformField.scaling(planes[0])
    if len(planes) != 4:
        raise IoError(path + ": quaternion field needs 4 planes")
    from .engine3d import rotation3d  # renormalizes like field.hpp:169-171
    return rotation3d(np.stack(planes, -1)[None])


# ------------------------------------------------------------------ XCF1

# "XCF1" | u8 group | i32 K | i32 n_radii | i32 n_angles | f64 r_max |
# f64 r_min | f64 r_domain | i64 n_rows | i64 n_cols | column-major complex<f64>
_XCF1_HEAD = struct.Struct("<4sBiiidddqq")


def retained_ks(K: int, n_periodic: int) -> list:
    """freq_filter.hpp:52-59."""
    kh = int(K) // 2
    if kh > n_periodic // 2:
        raise ValueError("band limit too large for sampling rate")
    return list(range(-kh, kh + 1))


def write_filter(path: str, f: FreqFilter2) -> None:
    """io.hpp:255-274."""
    comps = np.asarray(f.comps, np.complex128)
    head = _XCF1_HEAD.pack(b"XCF1", 0 if f.group == XformKind.rotation2 else 1, f.K, f.n_radii,
                           f.n_angles, float(f.r_max), float(f.r_min), float(f.r_domain),
                           comps.shape[0], comps.shape[1])
    body = np.ascontiguousarray(comps.T).astype("<c16").tobytes()  # column by column
    with _open_w(path) as out:
        out.write(head)
        out.write(body)


def read_filter(path: str) -> FreqFilter2:
    """io.hpp:276-316 (2D groups; a 3D container is rejected)."""
    data = _slurp(path)
    if len(data) < 4 or data[:4] != b"XCF1":
        raise IoError(path + ": not a filter container")
    if len(data) >= 5 and data[4] > 1:
        raise IoError(path + ": container holds a 3D filter")
    if len(data) < _XCF1_HEAD.size:
        raise IoError(path + ": truncated container")
    _, tag, K, n_radii, n_angles, r_max, r_min, r_domain, rows, cols = \
        _XCF1_HEAD.unpack_from(data)
    group = XformKind.rotation2 if tag == 0 else XformKind.scale2
    ks = retained_ks(K, n_angles if group == XformKind.rotation2 else n_radii)
    if cols != len(ks):
        raise IoError(path + ": component count does not match band limit")
    n = rows * cols
    if rows < 0 or len(data) < _XCF1_HEAD.size + 16 * n:
        raise IoError(path + ": truncated container")
    comps = np.frombuffer(data, "<c16", count=n, offset=_XCF1_HEAD.size).reshape(cols, rows).T
    return FreqFilter2(group, K, ks, comps.astype(np.complex128), n_radii, n_angles, r_max,
                       r_min, r_domain)


def write_filter3(path: str, f) -> None:
    """io.hpp:318-338: XCF1 with group tag 2, (K, n_radii, 0, r_max, 0, 0), then
    the (n_radii, (K+1)^2) coefficients column by column."""
    coeffs = np.asarray(f.coeffs, np.complex128)
    head = _XCF1_HEAD.pack(b"XCF1", 2, int(f.K), int(f.n_radii), 0, float(f.r_max), 0.0, 0.0,
                           coeffs.shape[0], coeffs.shape[1])
    with _open_w(path) as out:
        out.write(head)
        out.write(np.ascontiguousarray(coeffs.T).astype("<c16").tobytes())


def read_filter3(path: str):
    """io.hpp:340-368."""
    from .engine3d import SphFilter3
    data = _slurp(path)
    if len(data) < 4 or data[:4] != b"XCF1":
        raise IoError(path + ": not a filter container")
    if len(data) < 5 or data[4] != 2:
        raise IoError(path + ": not a 3D filter")
    if len(data) < _XCF1_HEAD.size:
        raise IoError(path + ": truncated container")
    _, _, K, n_radii, _, r_max, _, _, rows, cols = _XCF1_HEAD.unpack_from(data)
    if cols != (K + 1) * (K + 1):
        raise IoError(path + ": coefficient count does not match band limit")
    n = rows * cols
    if rows < 0 or len(data) < _XCF1_HEAD.size + 16 * n:
        raise IoError(path + ": truncated container")
    coeffs = np.frombuffer(data, "<c16", count=n, offset=_XCF1_HEAD.size).reshape(cols, rows).T
    return SphFilter3(K, n_radii, r_max, coeffs.astype(np.complex128))


__all__ = ["IoError", "read_pgm", "write_pgm", "write_pfm_planes", "read_pfm_planes",
           "write_pfm", "read_pfm_field", "write_xform", "read_xform", "write_filter",
           "read_filter", "retained_ks", "write_filter3", "read_filter3", "read_polylines_csv"]


def read_polylines_csv(path: str) -> list:
    """io.hpp:372-394: "x,y" rows, a blank line separates polylines."""
    try:
        f = open(path)
    except OSError:
        raise IoError("cannot open " + path) from None
    lines = [[]]
    with f:
        for row in f.read().split("\n"):
            if not row.strip(" \t\r"):
                if lines[-1]:
                    lines.append([])
                continue
            try:
                xs, ys = row.split(",", 1)
                lines[-1].append((float(xs), float(ys.split()[0] if ys.split() else ys)))
            except ValueError:
                raise IoError(path + ": bad polyline row: " + row) from None
    if not lines[-1]:
        lines.pop()
    if not lines:
        raise IoError(path + ": no polylines")
    return lines
