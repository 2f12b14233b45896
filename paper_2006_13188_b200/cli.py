"""Command-line surface of the reference (proj/tools/xconv_cli.cpp) over the
B200 path: the `xcorr`, `xconv`, `smooth`, `detect`, `contour`, `lic`, `decompose` and `steer3d`
subcommands with the reference's options, file formats (fileio.py), JSON
sidecars and exit codes.

    python -m paper_2006_13188_b200.cli xcorr --signal s.pfm --xform t.pfm \
        --filter f.xcf --output out.pfm

Exit codes (xconv_cli.cpp:1-4, 921-941): 0 success, 2 parameter error
(std::invalid_argument / bad options), 3 I/O error, 1 any other error.
Images are .pgm (8/16 bit) or .pfm (two planes = complex); 8-bit outputs are
min-max normalized with the mapping recorded in <output>.json.

Not carried over: `--method brute` and `oracle-check` run the reference's
dense brute-force oracle, which lives with the tests (oracle/) in this build;
`ecd`, `contours`, `lic` and `steer3d` are applications outside the hot path
(DESIGN.md section 9).
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

import numpy as np

from . import engine as E
from . import fileio as io


def _load_image(path: str) -> np.ndarray:
    """xconv_cli.cpp:33-37: .pgm (real) or .pfm (real or complex)."""
    if path.endswith(".pgm"):
        return io.read_pgm(path)
    if path.endswith(".pfm"):
        f = io.read_pfm_field(path)
        return np.real(f).copy() if not np.any(np.imag(f)) else f
    raise io.IoError("unsupported image format (want .pgm or .pfm): " + path)


def _save_image(path: str, f, sidecar: dict) -> None:
    """xconv_cli.cpp:39-56: .pfm raw; .pgm min-max normalized to 8 bits."""
    if path.endswith(".pfm"):
        io.write_pfm(path, f)
        return
    if not path.endswith(".pgm"):
        raise io.IoError("unsupported output format (want .pgm or .pfm): " + path)
    re = np.real(np.asarray(f)).astype(np.float64)
    lo, hi = float(re.min()), float(re.max())
    norm = (re - lo) / (hi - lo) if hi > lo else np.zeros_like(re)
    sidecar["normalization"] = {"min": lo, "max": hi, "maxval": 255}
    io.write_pgm(path, norm)


def _write_sidecar(image_path: str, sidecar: dict) -> None:
    """xconv_cli.cpp:58-64."""
    path = image_path + ".json"
    try:
        with open(path, "w") as out:
            out.write(json.dumps(sidecar, indent=2, sort_keys=True) + "\n")
    except OSError:
        raise io.IoError("cannot open " + path + " for writing") from None


def _parse_group(g: str) -> E.XformKind:
    """xconv_cli.cpp:66-71."""
    if g == "rotation":
        return E.XformKind.rotation2
    if g == "scale":
        return E.XformKind.scale2
    if g == "rotation3d":
        return E.XformKind.rotation3
    raise ValueError("--group must be rotation, scale, or rotation3d")


def _common(a) -> dict:
    return {"seed": a.seed, "threads": a.threads}


# ------------------------------------------------------------------ commands

def _load_engine_inputs(a):
    kind = _parse_group(a.group)
    H = _load_image(a.signal)
    T = io.read_xform(a.xform, kind)
    F = io.read_filter(a.filter)
    if F.group != kind:
        raise ValueError("--filter " + a.filter + " was decomposed for a different group")
    return kind, H, T, F


def cmd_engine(a, correlate: bool) -> int:
    """xconv_cli.cpp:233-286 (xcorr / xconv)."""
    if _parse_group(a.group) == E.XformKind.rotation3:
        raise ValueError("--group rotation3d: use the steer3d subcommand")
    if a.method != "fast":
        raise ValueError("--method brute: the dense brute-force oracle is test-side only "
                         "in the GPU build (oracle/)")
    _, H, T, F = _load_engine_inputs(a)
    t0 = time.perf_counter()
    r = (E.xcorr_fast if correlate else E.xconv_fast)(H, T, F)
    timings = {k: v for k, v in r.seconds.items() if k in ("render", "fft", "combine",
                                                          "premultiply")}
    timings["total"] = time.perf_counter() - t0
    sidecar = {"command": "xcorr" if correlate else "xconv",
               "parameters": {"signal": a.signal, "xform": a.xform, "filter": a.filter,
                              "group": a.group, "method": a.method, **_common(a)},
               "counters": {"standard-convolutions": r.standard_ops,
                            "components": F.n_components()},
               "timings": timings}
    _save_image(a.output, r.output, sidecar)
    _write_sidecar(a.output, sidecar)
    return 0


def cmd_smooth(a) -> int:
    """xconv_cli.cpp:288-330."""
    _, H, T, F = _load_engine_inputs(a)
    t0 = time.perf_counter()
    r = E.smooth_adaptive(H, T, F, not a.unnormalized)
    sidecar = {"command": "smooth",
               "parameters": {"signal": a.signal, "xform": a.xform, "filter": a.filter,
                              "group": a.group, "unnormalized": bool(a.unnormalized),
                              **_common(a)},
               "counters": {"standard-convolutions": r.standard_ops,
                            "clamped-pixels": r.clamped_pixels},
               "timings": {"total": time.perf_counter() - t0}}
    _save_image(a.output, r.output, sidecar)
    _write_sidecar(a.output, sidecar)
    return 0


def cmd_lic(a) -> int:
    """xconv_cli.cpp:602-639: seeded white noise smeared along a rotation field
    (lic.hpp:37-55 over the GPU path)."""
    from .lic import lic
    T = io.read_xform(a.field, E.XformKind.rotation2)
    t0 = time.perf_counter()
    out = lic(T, a.length, a.line_width, a.seed, not a.unnormalized, a.K)
    sidecar = {"command": "lic",
               "parameters": {"field": a.field, "length": a.length, "line-width": a.line_width,
                              "K": a.K, "unnormalized": bool(a.unnormalized), **_common(a)},
               "timings": {"total": time.perf_counter() - t0}}
    _save_image(a.output, out, sidecar)
    _write_sidecar(a.output, sidecar)
    return 0


def cmd_contour(a) -> int:
    """xconv_cli.cpp:527-599: complement matching of contour fragments; the
    match CSV holds x,y,angle,score rows (17 significant digits)."""
    from .contour import match_contours, rasterize_contours
    qlines = io.read_polylines_csv(a.query)
    tlines = io.read_polylines_csv(a.target)
    w, h = a.width, a.height
    if w <= 0 or h <= 0:
        mx = max(x for lines in (qlines, tlines) for ln in lines for x, _ in ln)
        my = max(y for lines in (qlines, tlines) for ln in lines for _, y in ln)
        mx, my = max(mx, 0.0), max(my, 0.0)
        if w <= 0:
            w = int(math.ceil(mx)) + 8
        if h <= 0:
            h = int(math.ceil(my)) + 8
    t0 = time.perf_counter()
    query = rasterize_contours(qlines, w, h, a.sigma)
    target = rasterize_contours(tlines, w, h, a.sigma)
    matches = match_contours(query, target, a.query_x, a.query_y, a.eps, a.K, a.top)
    try:
        with open(a.output, "w") as out:
            for m in matches:
                out.write(f"{m.x},{m.y},{m.angle:.17g},{m.score:.17g}\n")
    except OSError:
        raise io.IoError("cannot open " + a.output + " for writing") from None
    sidecar = {"command": "contour",
               "parameters": {"query": a.query, "target": a.target, "query-x": a.query_x,
                              "query-y": a.query_y, "eps": a.eps, "K": a.K, "width": w,
                              "height": h, "sigma": a.sigma, "top": a.top, **_common(a)},
               "counters": {"matches": len(matches)},
               "timings": {"total": time.perf_counter() - t0}}
    _write_sidecar(a.output, sidecar)
    return 0


def cmd_detect(a) -> int:
    """xconv_cli.cpp:348-405."""
    img = _load_image(a.image)
    pat = _load_image(a.pattern)
    ph, pw = pat.shape
    cx = a.center_x if a.center_x >= 0 else (pw - 1) / 2.0
    cy = a.center_y if a.center_y >= 0 else (ph - 1) / 2.0
    eps = a.eps if a.eps > 0 else min(pw, ph) / 2.0
    t0 = time.perf_counter()
    vf = E.build_optimal_filter(np.real(pat), cx, cy, eps)
    det = E.detect_pattern(np.real(img), vf, a.K)
    peaks = [{"x": p.x, "y": p.y, "value": p.value} for p in det.peaks]
    sidecar = {"command": "detect",
               "parameters": {"image": a.image, "pattern": a.pattern, "center-x": cx,
                              "center-y": cy, "eps": eps, "K": a.K, **_common(a)},
               "counters": {"standard-convolutions": det.standard_ops,
                            "peaks": len(det.peaks)},
               "peaks": peaks,
               "timings": {"total": time.perf_counter() - t0}}
    _save_image(a.output, det.response, sidecar)
    _write_sidecar(a.output, sidecar)
    if a.peaks_csv:
        try:
            with open(a.peaks_csv, "w") as out:
                for p in det.peaks:
                    out.write(f"{p.x},{p.y},{p.value:g}\n")
        except OSError:
            raise io.IoError("cannot open " + a.peaks_csv + " for writing") from None
    return 0


def _decompose3(a) -> int:
    """xconv_cli.cpp:739-780: a PFM stack of z slices -> SphFilter3 -> XCF1."""
    from . import engine3d as E3
    planes = io.read_pfm_planes(a.input)
    vol = np.stack([np.asarray(p, np.float64) for p in planes])  # (nz, h, w)
    nz, h, w = vol.shape
    cx = a.center_x if a.center_x >= 0 else (w - 1) / 2.0
    cy = a.center_y if a.center_y >= 0 else (h - 1) / 2.0
    cz = (nz - 1) / 2.0
    r_max = a.r_max if a.r_max > 0 else min(cx, cy, cz, w - 1 - cx, h - 1 - cy, nz - 1 - cz)
    if r_max <= 0:
        raise ValueError("--r-max must be positive (volume too small?)")
    n_radii = a.n_radii if a.n_radii > 0 else 2 * int(math.ceil(r_max))
    t0 = time.perf_counter()
    F = E3.decompose_rotation3(vol, cx, cy, cz, a.K, n_radii, r_max)
    io.write_filter3(a.output, F)
    sidecar = {"command": "decompose",
               "parameters": {"input": a.input, "group": a.group, "K": a.K, "center-x": cx,
                              "center-y": cy, "center-z": cz, "n-radii": n_radii,
                              "r-max": r_max, **_common(a)},
               "counters": {"steering-products": sum((2 * l + 1) ** 2 for l in range(F.K + 1))},
               "timings": {"total": time.perf_counter() - t0}}
    _write_sidecar(a.output, sidecar)
    return 0


def cmd_steer3d(a) -> int:
    """xconv_cli.cpp:645-688: rotate a 3D filter by a quaternion and write the
    reconstruction on the (2R+1)^3 grid as a PFM stack of z slices (real part)."""
    from . import engine3d as E3
    F = io.read_filter3(a.filter)
    q = np.asarray(a.quat, np.float64)
    nq = float(np.linalg.norm(q))
    if nq < 1e-12:
        raise ValueError("--quat must be a nonzero quaternion")
    q = q / nq
    t0 = time.perf_counter()
    rot = E3.steer_filter3(F, q)
    R = int(math.ceil(F.r_max))
    n = 2 * R + 1
    vol = E3.reconstruct3(rot, n, n, n, float(R), float(R), float(R))
    io.write_pfm_planes(a.output, [np.ascontiguousarray(vol[z].real) for z in range(n)])
    sidecar = {"command": "steer3d",
               "parameters": {"filter": a.filter, "quat": [float(v) for v in a.quat],
                              **_common(a)},
               "counters": {"degrees": F.K + 1,
                            "steering-products": sum((2 * l + 1) ** 2 for l in range(F.K + 1))},
               "timings": {"total": time.perf_counter() - t0}}
    _write_sidecar(a.output, sidecar)
    return 0


def cmd_decompose(a) -> int:
    """xconv_cli.cpp:690-829 (2D groups)."""
    kind = _parse_group(a.group)
    if kind == E.XformKind.rotation3:
        return _decompose3(a)
    img = _load_image(a.input)
    h, w = img.shape
    cx = a.center_x if a.center_x >= 0 else (w - 1) / 2.0
    cy = a.center_y if a.center_y >= 0 else (h - 1) / 2.0
    r_max = a.r_max if a.r_max > 0 else min(cx, cy, w - 1 - cx, h - 1 - cy)
    if r_max <= 0:
        raise ValueError("--r-max must be positive (image too small?)")
    n_radii = a.n_radii if a.n_radii > 0 else 2 * int(math.ceil(r_max))
    n_angles = a.n_angles if a.n_angles > 0 else max(32, 2 * a.K + 2)
    n_angles += n_angles % 2
    t0 = time.perf_counter()
    if kind == E.XformKind.rotation2:
        F = E.decompose_rotation2(img, cx, cy, a.K, n_radii, n_angles, r_max)
    else:
        F = E.decompose_scale2(img, cx, cy, a.K, n_radii, n_angles, a.r_min, r_max, a.r_domain)
    io.write_filter(a.output, F)
    R = int(math.ceil(F.r_max))
    if a.components_pfm:
        planes = []
        for ci in range(F.n_components()):
            comp = E.render_component(F, ci, 2 * R + 1, 2 * R + 1, float(R), float(R))
            planes += [np.real(comp), np.imag(comp)]
        io.write_pfm_planes(a.components_pfm, planes)
    sidecar = {"command": "decompose",
               "parameters": {"input": a.input, "group": a.group, "K": a.K, "center-x": cx,
                              "center-y": cy, "n-radii": n_radii, "n-angles": n_angles,
                              "r-min": a.r_min, "r-max": r_max, "r-domain": F.domain_top(),
                              **_common(a)},
               "counters": {"components": F.n_components()},
               "timings": {"total": time.perf_counter() - t0}}
    if a.recon:
        recon = E.reconstruct(F, 2 * R + 1, 2 * R + 1, float(R), float(R))
        _save_image(a.recon, recon, sidecar)
    _write_sidecar(a.output, sidecar)
    return 0


# ------------------------------------------------------------------ parser

def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="xconv",
        description="Spatially-adaptive filtering on B200: extended correlation/convolution "
                    "with per-pixel rotated or scaled filters, smoothing, detection and "
                    "filter decomposition.")
    # --seed / --threads are accepted before or after the subcommand (CLI11
    # fallthrough, xconv_cli.cpp:221-230)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--threads", type=int, default=1)
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--seed", type=int, default=argparse.SUPPRESS)
    common.add_argument("--threads", type=int, default=argparse.SUPPRESS)
    sub = ap.add_subparsers(dest="command", required=True)
    for name in ("xcorr", "xconv"):
        c = sub.add_parser(name, parents=[common])
        c.add_argument("--signal", required=True)
        c.add_argument("--xform", required=True)
        c.add_argument("--filter", required=True)
        c.add_argument("--group", default="rotation")
        c.add_argument("--method", default="fast", choices=["fast", "brute"])
        c.add_argument("--output", required=True)
    c = sub.add_parser("smooth", parents=[common])
    c.add_argument("--signal", required=True)
    c.add_argument("--xform", required=True)
    c.add_argument("--filter", required=True)
    c.add_argument("--group", default="rotation")
    c.add_argument("--unnormalized", action="store_true")
    c.add_argument("--output", required=True)
    c = sub.add_parser("detect", parents=[common])
    c.add_argument("--image", required=True)
    c.add_argument("--pattern", required=True)
    c.add_argument("--center-x", type=float, default=-1.0)
    c.add_argument("--center-y", type=float, default=-1.0)
    c.add_argument("--eps", type=float, default=0.0)
    c.add_argument("--K", type=int, default=16)
    c.add_argument("--output", required=True)
    c.add_argument("--peaks-csv", default="")
    c = sub.add_parser("contour", parents=[common])
    c.add_argument("--query", required=True)
    c.add_argument("--target", required=True)
    c.add_argument("--query-x", type=float, required=True)
    c.add_argument("--query-y", type=float, required=True)
    c.add_argument("--eps", type=float, default=8.0)
    c.add_argument("--K", type=int, default=16)
    c.add_argument("--width", type=int, default=0)
    c.add_argument("--height", type=int, default=0)
    c.add_argument("--sigma", type=float, default=1.5)
    c.add_argument("--top", type=int, default=9)
    c.add_argument("--output", required=True)
    c = sub.add_parser("lic", parents=[common])
    c.add_argument("--field", required=True)
    c.add_argument("--length", type=float, default=8.0)
    c.add_argument("--line-width", type=float, default=1.2)
    c.add_argument("--K", type=int, default=16)
    c.add_argument("--unnormalized", action="store_true")
    c.add_argument("--output", required=True)
    c = sub.add_parser("steer3d", parents=[common])
    c.add_argument("--filter", required=True)
    c.add_argument("--quat", type=float, nargs=4, default=[1.0, 0.0, 0.0, 0.0])
    c.add_argument("--output", required=True)
    c = sub.add_parser("decompose", parents=[common])
    c.add_argument("--input", required=True)
    c.add_argument("--group", default="rotation")
    c.add_argument("--K", type=int, default=16)
    c.add_argument("--center-x", type=float, default=-1.0)
    c.add_argument("--center-y", type=float, default=-1.0)
    c.add_argument("--n-radii", type=int, default=0)
    c.add_argument("--n-angles", type=int, default=0)
    c.add_argument("--r-min", type=float, default=1.0)
    c.add_argument("--r-max", type=float, default=0.0)
    c.add_argument("--r-domain", type=float, default=0.0)
    c.add_argument("--output", required=True)
    c.add_argument("--components-pfm", default="")
    c.add_argument("--recon", default="")
    return ap


def main(argv=None) -> int:
    ap = _parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # bad options: CLI11 parse error -> 2
        return 0 if e.code == 0 else 2
    try:
        return {"xcorr": lambda: cmd_engine(a, True), "xconv": lambda: cmd_engine(a, False),
                "smooth": lambda: cmd_smooth(a), "detect": lambda: cmd_detect(a),
                "decompose": lambda: cmd_decompose(a), "lic": lambda: cmd_lic(a),
                "contour": lambda: cmd_contour(a),
                "steer3d": lambda: cmd_steer3d(a)}[a.command]()
    except io.IoError as e:
        print(f"io error: {e}", file=sys.stderr)
        return 3
    except ValueError as e:
        print(f"parameter error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 (the reference's catch-all, exit 1)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
