"""Contour matching over the GPU path (contour.hpp:8-189; the SURVEY 8(b)
caller match_contours).  CPU: blur and rasterization against the restatement
and test_contour.cpp:90-107; GPU: test_contour.cpp:43-88 and the scatter
response / peak list against the oracle composition."""
import math

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import contour as CT

TOL = 1e-5


def fracture_curve(cx, cy, half_len):  # test_contour.cpp:12-17
    t = np.arange(-half_len, half_len + 1e-9, 0.5)
    return [(cx + v, cy + 2.5 * math.sin(0.35 * v) + 1.2 * math.cos(0.8 * v)) for v in t]


def blob_arc(cx, cy, a0, a1, steps):  # test_contour.cpp:20-28
    out = []
    for i in range(steps + 1):
        a = a0 + (a1 - a0) * i / steps
        r = 18 + 3 * math.sin(2 * a) + 2 * math.cos(3 * a)
        out.append((cx + r * math.cos(a), cy + r * math.sin(a)))
    return out


def translated(c, tx, ty):
    return [(x + tx, y + ty) for x, y in c]


# ------------------------------------------------------------------ CPU

def test_blur_matches_oracle(orc):
    r = np.random.default_rng(3)
    img = r.random((23, 31))
    for s in (0.3, 1.5, 2.0, 4.0):
        assert np.abs(CT.gaussian_blur(img, s) - orc.gaussian_blur(img, s)).max() < 1e-13


def test_rasterization_nonnegative_with_normals_on_the_curve():  # test_contour.cpp:98-107
    n = 48
    s = X.rasterize_contours([[(10, 24), (38, 24)]], n, n)
    assert (s.signal >= 0).all()
    for x in range(16, 33, 4):
        assert s.coverage[24, x] > 0.1
        assert abs(float(CT.normalize_angle(s.normal_angle[24, x] + math.pi / 2))) < 1e-6


def test_empty_query_region_rejected():  # test_contour.cpp:90-96
    n = 48
    scene = X.rasterize_contours([[(4, 8), (44, 8)]], n, n)
    with pytest.raises(ValueError, match="empty contour region"):
        X.match_contours(scene, scene, 30.0, 40.0, 4.0, 8)


# ------------------------------------------------------------------ GPU

def _split_shape():
    n, cx, cy = 80, 40.0, 40.0
    frac = fracture_curve(cx, cy, 17)
    upper = blob_arc(cx, cy, math.pi, 2 * math.pi, 64)
    lower = blob_arc(cx, cy, 0.0, math.pi, 64)
    tx, ty = 4.0, -3.0
    query = X.rasterize_contours([upper, frac], n, n)
    target = X.rasterize_contours([translated(lower, tx, ty),
                                   translated(frac[::-1], tx, ty)], n, n)
    return query, target, cx, cy + 1.0, tx, ty


@pytest.mark.gpu
def test_complement_halves_match_at_the_true_placement():  # test_contour.cpp:43-71
    query, target, qx, qy, tx, ty = _split_shape()
    m = X.match_contours(query, target, qx, qy, 8.0, 16)
    assert m
    top = m[0]
    assert math.hypot(top.x - (qx + tx), top.y - (qy + ty)) <= 2.0
    assert abs(float(CT.normalize_angle(top.angle))) <= 3.0 * math.pi / 180
    self_m = X.match_contours(query, query, qx, qy, 8.0, 16)
    assert self_m and self_m[0].score < top.score


@pytest.mark.gpu
def test_straight_edges_align_antiparallel(orc):  # test_contour.cpp:73-88
    n = 64
    query = X.rasterize_contours([[(8, 32), (56, 32)]], n, n)
    target = X.rasterize_contours([[(56, 40), (8, 40)]], n, n)
    m = X.match_contours(query, target, 32.0, 32.0, 8.0, 16)
    assert m
    assert abs(m[0].y - 40) <= 2
    assert orc.orientation_distance(m[0].angle, 0.0) <= 3.0 * math.pi / 180


@pytest.mark.gpu
def test_scatter_response_and_peaks_match_oracle(orc):
    """The GPU part of match_contours (contour.hpp:156-169) against the oracle
    composition on the same vote filter: response within 1e-5, peaks exact."""
    query, target, qx, qy, _, _ = _split_shape()
    eps, K = 8.0, 16
    frame = CT.normalize_angle(query.normal_angle + math.pi)
    vf = X.build_vote_filter(query.signal, frame, qx, qy, eps)
    w_o, R_o = orc.build_vote_filter(query.signal, frame, qx, qy, eps)
    assert R_o == vf.radius and np.abs(np.asarray(w_o) - vf.weights).max() < 1e-12
    R = vf.radius
    n_radii, n_angles = max(4, 2 * R), max(32, 8 * ((R + 3) // 4) * 4)
    F = X.decompose_rotation2(vf.weights, float(R), float(R), K, n_radii, n_angles, R + 0.5)
    Fo = orc.decompose_rotation2(vf.weights, float(R), float(R), K, n_radii, n_angles, R + 0.5)
    got = X.xconv_fast(target.signal, X.XformField.rotation(target.normal_angle), F).output.real
    ref = orc.xconv_fast(target.signal, 0, target.normal_angle, Fo)[0].real
    assert orc.rel_l2(got, ref) < TOL
    pg = X.find_peaks(np.ascontiguousarray(got, np.float64), eps / 2, 0.1)
    po = orc.find_peaks(ref, eps / 2, 0.1)
    assert [(p.x, p.y) for p in pg[:3]] == [(int(x), int(y)) for x, y, *_ in po[:3]]


def test_polyline_csv(tmp_path):  # io.hpp:372-394
    from paper_2006_13188_b200 import fileio as io
    p = tmp_path / "c.csv"
    p.write_text("1,2\n3.5,4\n\n  \n5,6\n7,8\n9,10\n\n")
    assert io.read_polylines_csv(str(p)) == [[(1.0, 2.0), (3.5, 4.0)],
                                             [(5.0, 6.0), (7.0, 8.0), (9.0, 10.0)]]
    p.write_text("1;2\n")
    with pytest.raises(io.IoError, match="bad polyline row"):
        io.read_polylines_csv(str(p))
    p.write_text("\n\n")
    with pytest.raises(io.IoError, match="no polylines"):
        io.read_polylines_csv(str(p))


@pytest.mark.gpu
def test_cli_contour_matches_api(tmp_path):  # xconv_cli.cpp:527-599
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    q, t = [[(8, 32), (56, 32)]], [[(56, 40), (8, 40)]]
    for name, lines in (("q.csv", q), ("t.csv", t)):
        (tmp_path / name).write_text("\n\n".join("\n".join(f"{x},{y}" for x, y in ln)
                                                 for ln in lines) + "\n")
    out = str(tmp_path / "m.csv")
    r = subprocess.run([sys.executable, "-m", "paper_2006_13188_b200", "contour", "--query",
                        str(tmp_path / "q.csv"), "--target", str(tmp_path / "t.csv"),
                        "--query-x", "32", "--query-y", "32", "--width", "64", "--height", "64",
                        "--output", out], cwd=root, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = [ln.split(",") for ln in open(out).read().split()]
    api = X.match_contours(X.rasterize_contours(q, 64, 64), X.rasterize_contours(t, 64, 64),
                           32.0, 32.0, 8.0, 16)
    assert len(rows) == len(api) > 0
    assert (int(rows[0][0]), int(rows[0][1])) == (api[0].x, api[0].y)
    assert float(rows[0][2]) == api[0].angle and float(rows[0][3]) == api[0].score
    side = json.load(open(out + ".json"))
    assert side["command"] == "contour" and side["counters"]["matches"] == len(api)
