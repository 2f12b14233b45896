"""File formats and CLI: ports of proj/tests/test_io.cpp, byte
layouts pinned against io.hpp, and the CLI's exit codes and sidecars
(xconv_cli.cpp).  CPU only except the GPU-marked CLI runs at the end."""
import json
import struct

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import cli
from paper_2006_13188_b200 import fileio as io


# ---------------------------------------------------------------- test_io.cpp ports

def test_pgm_round_trip_8_and_16_bit(tmp_path):  # test_io.cpp:22-36
    f = np.random.default_rng(31).random((9, 13))
    for maxval in (255, 65535):
        p = str(tmp_path / "t.pgm")
        io.write_pgm(p, f, maxval)
        g = io.read_pgm(p)
        assert g.shape == (9, 13)
        assert np.abs(g - f).max() < 0.5 / maxval + 1e-12


def test_pgm_rejects_bad_headers_and_truncated_rasters(tmp_path):  # test_io.cpp:38-51
    p = tmp_path / "bad.pgm"
    p.write_bytes(b"P6\n2 2\n255\nxxxx")
    with pytest.raises(io.IoError):
        io.read_pgm(str(p))
    p.write_bytes(b"P5\n4 4\n255\nxx")
    with pytest.raises(io.IoError, match="truncated PGM raster"):
        io.read_pgm(str(p))
    with pytest.raises(io.IoError, match="cannot open"):
        io.read_pgm("/nonexistent/xconv.pgm")


def test_pgm_header_comments_and_16_bit_big_endian(tmp_path):  # io.hpp:20-32, 72-78
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# comment\n2 # w\n1\n65535\n\x01\x02\xff\xff")
    g = io.read_pgm(str(p))
    assert g.shape == (1, 2)
    assert g[0, 0] == 0x0102 / 65535 and g[0, 1] == 1.0


def test_pgm_write_rounds_and_clamps(tmp_path):  # io.hpp:83-103 (std::lround, clamp)
    p = str(tmp_path / "r.pgm")
    io.write_pgm(p, np.array([[-1.0, 0.5 / 255, 1.5 / 255, 2.0]]))
    assert open(p, "rb").read() == b"P5\n4 1\n255\n" + bytes([0, 1, 2, 255])


def test_pfm_round_trip_real_and_complex(tmp_path):  # test_io.cpp:53-66
    rng = np.random.default_rng(32)
    p = str(tmp_path / "t.pfm")
    re = rng.uniform(-1, 1, (5, 7))
    io.write_pfm(p, re)
    re2 = io.read_pfm_field(p)
    assert np.linalg.norm(re2 - re) / np.linalg.norm(re) < 1e-6
    assert not np.any(np.imag(re2))
    cx = rng.uniform(-1, 1, (8, 6)) + 1j * rng.uniform(-1, 1, (8, 6))
    io.write_pfm(p, cx)
    cx2 = io.read_pfm_field(p)
    assert np.linalg.norm(cx2 - cx) / np.linalg.norm(cx) < 1e-6
    assert len(io.read_pfm_planes(p)) == 2


def test_pfm_byte_layout(tmp_path):  # io.hpp:112-129: header, LE fp32, rows bottom-up
    p = str(tmp_path / "l.pfm")
    io.write_pfm_planes(p, [np.array([[1.0, 2.0], [3.0, 4.0]])])
    want = b"Pf\n2 2\n-1.0\n" + struct.pack("<4f", 3.0, 4.0, 1.0, 2.0)
    assert open(p, "rb").read() == want


def test_pfm_big_endian_plane_is_read(tmp_path):  # io.hpp:142-155 (positive scale)
    p = tmp_path / "be.pfm"
    p.write_bytes(b"Pf\n2 1\n1.0\n" + struct.pack(">2f", 0.25, -8.0))
    assert io.read_pfm_planes(str(p))[0].tolist() == [[0.25, -8.0]]
    p.write_bytes(b"PF\n2 1\n-1.0\n")
    with pytest.raises(io.IoError, match="expected grayscale Pf plane"):
        io.read_pfm_planes(str(p))
    p.write_bytes(b"Pf\n2 2\n-1.0\n" + b"\0" * 8)
    with pytest.raises(io.IoError, match="truncated PFM raster"):
        io.read_pfm_planes(str(p))


def test_pfm_round_trip_transformation_fields(tmp_path):  # test_io.cpp:68-93
    rng = np.random.default_rng(33)
    p = str(tmp_path / "x.pfm")
    ang = rng.uniform(-np.pi, np.pi, (4, 6))
    io.write_xform(p, X.XformField.rotation(ang))
    rot2 = io.read_xform(p, X.XformKind.rotation2)
    assert np.abs(rot2.angle - ang).max() < 1e-6
    sc = np.exp(rng.uniform(np.log(0.5), np.log(2.0), (7, 5)))
    io.write_xform(p, X.XformField.scaling(sc))
    sc2 = io.read_xform(p, X.XformKind.scale2)
    assert np.abs(sc2.scale - sc).max() < 1e-6
    from paper_2006_13188_b200 import engine3d as E3
    q = rng.normal(size=(1, 3, 4, 4))  # (nz, ny, nx, 4): the engine's layout
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    io.write_xform(p, E3.rotation3d(q))
    q2 = io.read_xform(p, X.XformKind.rotation3)
    assert q2.values.shape == (1, 3, 4, 4)
    assert np.abs(q2.values - q).max() < 1e-6
    # non-unit quaternions read back renormalized (field.hpp:169-171)
    io.write_xform(p, X.XformField(X.XformKind.rotation3, 2.0 * q))
    q3 = io.read_xform(p, X.XformKind.rotation3)
    assert np.abs(q3.values - q).max() < 1e-6
    with pytest.raises(io.IoError, match="single-slice"):
        io.write_xform(p, X.XformField(X.XformKind.rotation3, np.concatenate([q, q])))
    with pytest.raises(io.IoError, match="rotation field needs 1 plane"):
        io.read_xform(p, X.XformKind.rotation2)


def test_rotation_field_is_written_normalized(tmp_path):  # io.hpp:188-189, field.hpp:122-127
    p = str(tmp_path / "n.pfm")
    io.write_xform(p, X.XformField.rotation(np.array([[3 * np.pi, -np.pi / 2, 7.0]])))
    got = io.read_pfm_planes(p)[0][0]
    assert np.allclose(got, [-np.pi, -np.pi / 2, 7.0 - 2 * np.pi], atol=1e-6)


def _smooth_filter(R, seed):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[-R:R + 1, -R:R + 1]
    v = np.zeros(x.shape)
    for _ in range(6):
        bx, by, a, s = rng.uniform(-0.5, 0.5) * R, rng.uniform(-0.5, 0.5) * R, \
            rng.uniform(-1, 1), 1.2 + 0.8 * rng.random()
        v += a * np.exp(-((x - bx) ** 2 + (y - by) ** 2) / (2 * s * s))
    return v * np.exp(-(x * x + y * y) / (2 * (0.35 * R) ** 2))


def test_filter_container_round_trip_both_groups(tmp_path):  # test_io.cpp:95-122
    R = 5
    filt = _smooth_filter(R, 34)
    p = str(tmp_path / "f.xcf")
    rot = X.decompose_rotation2(filt, R, R, 6, 2 * R, 32, float(R))
    io.write_filter(p, rot)
    rot2 = io.read_filter(p)
    assert rot2.group == X.XformKind.rotation2 and rot2.K == rot.K
    assert list(rot2.ks) == list(rot.ks)
    assert np.abs(rot2.comps - rot.comps).max() == 0.0
    assert rot2.r_max == rot.r_max
    sc = X.decompose_scale2(filt, R, R, 8, 24, 16, 0.5, float(R), R + 2.0)
    io.write_filter(p, sc)
    sc2 = io.read_filter(p)
    assert sc2.group == X.XformKind.scale2
    assert sc2.r_min == sc.r_min and sc2.r_domain == sc.r_domain
    assert sc2.domain_top() == sc.domain_top()
    assert np.abs(sc2.comps - sc.comps).max() == 0.0


def test_filter_container_byte_layout(tmp_path):  # io.hpp:238-274
    F = X.FreqFilter2(X.XformKind.scale2, 2, [-1, 0, 1],
                      np.array([[1 + 2j, 3 + 4j, 5 + 6j], [7 + 8j, 9 + 10j, 11 + 12j]]),
                      4, 2, 3.0, 0.5, 3.5)
    p = str(tmp_path / "b.xcf")
    io.write_filter(p, F)
    want = b"XCF1" + struct.pack("<B", 1) + struct.pack("<iii", 2, 4, 2) + \
        struct.pack("<ddd", 3.0, 0.5, 3.5) + struct.pack("<qq", 2, 3) + \
        struct.pack("<12d", 1, 2, 7, 8, 3, 4, 9, 10, 5, 6, 11, 12)  # column-major
    assert open(p, "rb").read() == want


def test_filter_container_rejects_corrupt_and_3d(tmp_path):  # test_io.cpp:124-157
    p = tmp_path / "c.xcf"
    p.write_bytes(b"NOPE")
    with pytest.raises(io.IoError, match="not a filter container"):
        io.read_filter(str(p))
    p.write_bytes(b"XCF1" + struct.pack("<B", 2) + b"\0" * 60)
    with pytest.raises(io.IoError, match="container holds a 3D filter"):
        io.read_filter(str(p))
    F = X.FreqFilter2(X.XformKind.rotation2, 2, [-1, 0, 1], np.ones((3, 3)), 3, 8, 2.0)
    io.write_filter(str(p), F)
    data = p.read_bytes()
    p.write_bytes(data[:-5])
    with pytest.raises(io.IoError, match="truncated container"):
        io.read_filter(str(p))
    # column count must match the band limit (io.hpp:297-299)
    p.write_bytes(data[:5] + struct.pack("<i", 4) + data[9:])  # K = 4: 5 bands, 3 columns
    with pytest.raises(io.IoError, match="component count does not match band limit"):
        io.read_filter(str(p))


# ---------------------------------------------------------------- CLI (host-only paths)

def test_cli_decompose_writes_container_sidecar_and_components(tmp_path):
    R = 6
    img = tmp_path / "filt.pfm"
    io.write_pfm(str(img), _smooth_filter(R, 7))
    out, comps, recon = tmp_path / "f.xcf", tmp_path / "c.pfm", tmp_path / "r.pgm"
    rc = cli.main(["decompose", "--input", str(img), "--K", "8", "--output", str(out),
                   "--components-pfm", str(comps), "--recon", str(recon)])
    assert rc == 0
    F = io.read_filter(str(out))
    assert F.group == X.XformKind.rotation2 and F.n_components() == 9
    # the reference defaults: centre (w-1)/2, r_max fits the image, n_radii 2 ceil(r_max),
    # n_angles max(32, 2K+2) rounded up to even (xconv_cli.cpp:790-802)
    assert (F.r_max, F.n_radii, F.n_angles) == (6.0, 12, 32)
    ref = X.decompose_rotation2(io.read_pfm_field(str(img)), 6.0, 6.0, 8, 12, 32, 6.0)
    assert np.abs(F.comps - ref.comps).max() < 1e-12
    side = json.load(open(str(out) + ".json"))
    assert side["command"] == "decompose" and side["counters"]["components"] == 9
    assert side["parameters"]["n-angles"] == 32 and "normalization" in side
    assert len(io.read_pfm_planes(str(comps))) == 18
    assert io.read_pgm(str(recon)).shape == (13, 13)


def test_cli_exit_codes(tmp_path, capsys):  # xconv_cli.cpp:921-941
    assert cli.main(["xcorr", "--signal", "/nonexistent.pfm", "--xform", "x.pfm",
                     "--filter", "f.xcf", "--output", "o.pfm"]) == 3
    assert "io error" in capsys.readouterr().err
    assert cli.main(["xcorr", "--signal", "s.png", "--xform", "x.pfm", "--filter", "f.xcf",
                     "--output", "o.pfm"]) == 3  # unsupported image format
    assert cli.main(["xcorr", "--signal", "s.pfm"]) == 2  # missing required options
    assert cli.main(["nosuch"]) == 2
    # group mismatch between --group and the container (xconv_cli.cpp:262-264)
    s, x, f = tmp_path / "s.pfm", tmp_path / "x.pfm", tmp_path / "f.xcf"
    io.write_pfm(str(s), np.zeros((4, 4)))
    io.write_xform(str(x), X.XformField.scaling(np.ones((4, 4))))
    io.write_filter(str(f), X.FreqFilter2(X.XformKind.rotation2, 2, [-1, 0, 1],
                                         np.ones((3, 3)), 3, 8, 2.0))
    assert cli.main(["xconv", "--signal", str(s), "--xform", str(x), "--filter", str(f),
                     "--group", "scale", "--output", str(tmp_path / "o.pfm")]) == 2
    assert "was decomposed for a different group" in capsys.readouterr().err
    assert cli.main(["xcorr", "--signal", str(s), "--xform", str(x), "--filter", str(f),
                     "--group", "rotation3d", "--output", str(tmp_path / "o.pfm")]) == 2
    assert cli.main(["smooth", "--signal", str(s), "--xform", str(x), "--filter", str(f),
                     "--group", "bogus", "--output", str(tmp_path / "o.pfm")]) == 2
    assert cli.main(["--seed", "3", "decompose", "--input", str(s), "--r-max", "-1",
                     "--center-x", "0", "--output", str(f)]) == 2


# ---------------------------------------------------------------- CLI on the GPU

@pytest.mark.gpu
def test_cli_xcorr_xconv_smooth_match_oracle(tmp_path, orc):
    rng = np.random.default_rng(5)
    H, W, R = 40, 33, 6
    sig = rng.random((H, W))
    ang = rng.uniform(-np.pi, np.pi, (H, W))
    s, x, f = str(tmp_path / "s.pfm"), str(tmp_path / "x.pfm"), str(tmp_path / "f.xcf")
    io.write_pfm(s, sig)
    io.write_xform(x, X.XformField.rotation(ang))
    F = X.decompose_rotation2(_smooth_filter(R, 9), R, R, 8, 12, 32, float(R))
    io.write_filter(f, F)
    # the CLI reads fp32 files: the oracle sees exactly those values
    sig32 = io.read_pfm_field(s).real
    ang32 = io.read_xform(x, X.XformKind.rotation2).values
    OF = orc.Filter(0, F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max)
    for cmd, fn in (("xcorr", orc.xcorr_fast), ("xconv", orc.xconv_fast)):
        o = str(tmp_path / f"{cmd}.pfm")
        assert cli.main([cmd, "--signal", s, "--xform", x, "--filter", f, "--output", o]) == 0
        got = io.read_pfm_field(o)
        ref = fn(sig32, 0, ang32, OF)[0]
        assert orc.rel_l2(got, ref) < 1e-5
        side = json.load(open(o + ".json"))
        assert side["counters"] == {"standard-convolutions": 9, "components": 9}
        assert {"render", "fft", "combine", "total"} <= set(side["timings"])
    o = str(tmp_path / "sm.pgm")
    assert cli.main(["smooth", "--signal", s, "--xform", x, "--filter", f, "--output", o]) == 0
    side = json.load(open(o + ".json"))
    assert side["counters"]["standard-convolutions"] == 18
    ref = orc.smooth_adaptive(sig32, 0, ang32, OF, True)[0]
    lo, hi = side["normalization"]["min"], side["normalization"]["max"]
    assert abs(lo - ref.min()) < 1e-5 * abs(ref).max() and abs(hi - ref.max()) < 1e-5 * abs(ref).max()
    assert np.abs(io.read_pgm(o) - (ref - lo) / (hi - lo)).max() <= 0.5 / 255 + 1e-5


@pytest.mark.gpu
def test_cli_detect_matches_api(tmp_path):
    """xconv_cli.cpp:348-405: `detect` writes the vote response, a sidecar with the
    peaks, and the peaks CSV; the peaks equal detect_pattern's on the same inputs."""
    from paper_2006_13188_b200.workloads import paste_rotated
    R = 8
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    pat = np.exp(-((x - 2) ** 2 + (y + 1) ** 2) / 4.0) - 0.7 * np.exp(-((x + 3) ** 2 + y ** 2) / 3.0)
    img = np.zeros((96, 110))
    paste_rotated(img, pat, 30.0, 40.0, 0.6)
    paste_rotated(img, pat, 75.0, 62.0, -1.9)
    img += np.random.default_rng(4).normal(0, 0.01, img.shape)
    p_img, p_pat = str(tmp_path / "img.pfm"), str(tmp_path / "pat.pfm")
    io.write_pfm(p_img, img)
    io.write_pfm(p_pat, pat)
    out, csvp = str(tmp_path / "resp.pfm"), str(tmp_path / "peaks.csv")
    assert cli.main(["detect", "--image", p_img, "--pattern", p_pat, "--K", "12", "--output", out,
                     "--peaks-csv", csvp]) == 0
    img32, pat32 = io.read_pfm_field(p_img).real, io.read_pfm_field(p_pat).real
    # the CLI's defaults: centre (w-1)/2, eps = min(w, h)/2 (xconv_cli.cpp:374-377)
    vf = X.build_optimal_filter(pat32, R, R, (2 * R + 1) / 2.0)
    det = X.detect_pattern(img32, vf, 12)
    side = json.load(open(out + ".json"))
    assert side["counters"]["peaks"] == len(det.peaks) >= 2
    assert [(p["x"], p["y"]) for p in side["peaks"]] == [(p.x, p.y) for p in det.peaks]
    rows = [l.split(",") for l in open(csvp).read().split()]
    assert [(int(a), int(b)) for a, b, _ in rows] == [(p.x, p.y) for p in det.peaks]
    resp = io.read_pfm_field(out).real
    assert np.abs(resp - det.response).max() <= 1e-6 * np.abs(det.response).max()
