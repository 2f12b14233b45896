"""Line integral convolution (lic.hpp:9-55, acceptance
criterion 12) over the GPU path.  CPU: the seeded noise (bit-exact against the
oracle restatement and the std::mt19937_64 known answer), the kernel and the
parameter validation (test_lic.cpp:85-92).  GPU: parity with the oracle
composition (relative L2 <= 1e-5) and the reference's structure tests
(test_lic.cpp:20-83)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2006_13188_b200 as X

TOL = 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def circular_field(n):  # test_lic.cpp:9-16
    c = (n - 1) / 2.0
    y, x = np.mgrid[0:n, 0:n].astype(np.float64)
    return np.arctan2(y - c, x - c) + np.pi / 2


# ------------------------------------------------------------------ CPU

def test_white_noise_bit_exact(orc):
    for seed, (w, h) in ((42, (13, 7)), (7, (5, 9)), (2**63 + 5, (4, 4))):
        a = X.white_noise(w, h, seed)
        assert a.shape == (h, w)
        assert np.array_equal(a, orc.white_noise(w, h, seed))
        assert np.all((a >= 0) & (a < 1))
    # the C++ standard's check value: the 10000th output of a default-seeded
    # std::mt19937_64 is 9981545732273789042
    v = X.white_noise(10000, 1, 5489)[0, -1]
    assert v == (9981545732273789042 >> 11) * 2.0 ** -53
    assert not np.array_equal(X.white_noise(8, 8, 43), X.white_noise(8, 8, 42))


def test_anisotropic_gaussian_matches_oracle(orc):
    for length, width in ((8.0, 1.2), (6.0, 1.2), (5.0, 1.0), (2.3, 0.7)):
        a = X.anisotropic_gaussian(length, width)
        b = orc.anisotropic_gaussian(length, width)
        R = int(np.ceil(2.5 * length))
        assert a.shape == (2 * R + 1, 2 * R + 1)
        assert np.abs(a - b).max() < 1e-15
        assert a[R, R] == 1.0 and a[R, 0] > a[0, R]  # oriented along +x


def test_lic_parameter_validation():  # test_lic.cpp:85-92
    n = 16
    with pytest.raises(ValueError, match="lic needs a rotation2 field"):
        X.lic(X.XformField.scaling(np.ones((n, n))), 5.0, 1.0, 1)
    rot = X.XformField.rotation(np.zeros((n, n)))
    with pytest.raises(ValueError, match="need length > width > 0"):
        X.lic(rot, 1.0, 2.0, 1)
    with pytest.raises(ValueError, match="need length > width > 0"):
        X.lic(rot, 2.0, 0.0, 1)


# ------------------------------------------------------------------ GPU

def _mean_deviation(orc, out, sigma, target, keep_coh, mask=None):
    o, coh = orc.structure_tensor(out, sigma)
    sel = coh >= keep_coh
    if mask is not None:
        sel &= mask
    d = orc.orientation_distance(o[sel], np.broadcast_to(target, o.shape)[sel])
    return float(d.mean()) if d.size else np.inf, int(d.size)


@pytest.mark.gpu
@pytest.mark.parametrize("normalized", [True, False])
def test_lic_matches_oracle(orc, normalized):
    n = 48
    ang = circular_field(n)
    got = X.lic(X.XformField.rotation(ang), 5.0, 1.0, 42, normalized)
    ref = orc.lic(ang, 5.0, 1.0, 42, normalized)
    assert got.shape == (n, n)
    assert orc.rel_l2(got, ref) < TOL


@pytest.mark.gpu
def test_constant_field_renders_horizontal_streaks(orc):  # test_lic.cpp:20-34
    n = 96
    out = X.lic(X.XformField.rotation(np.zeros((n, n))), 8.0, 1.2, 5)
    inner = np.zeros((n, n), bool)
    inner[8:n - 8, 8:n - 8] = True
    dev, cnt = _mean_deviation(orc, out, 3.0, 0.0, 0.7, inner)
    assert cnt > 100
    assert dev < 5.0 * np.pi / 180


@pytest.mark.gpu
def test_circular_field_streaks_follow_the_field(orc):  # test_lic.cpp:36-56, criterion 12
    n = 128
    ang = circular_field(n)
    T = X.XformField.rotation(ang)
    out = X.lic(T, 6.0, 1.2, 7)
    c = (n - 1) / 2.0
    y, x = np.mgrid[0:n, 0:n]
    r = np.hypot(x - c, y - c)
    dev, cnt = _mean_deviation(orc, out, 2.0, T.angle, 0.3, (r >= 16) & (r <= 56))
    assert cnt > 1000
    assert dev < 15.0 * np.pi / 180
    assert np.array_equal(X.lic(T, 6.0, 1.2, 7), out)  # repeat runs are bit-identical


@pytest.mark.gpu
def test_seeds_and_unnormalized_variant(orc):  # test_lic.cpp:58-83
    T = X.XformField.rotation(circular_field(48))
    a = X.lic(T, 5.0, 1.0, 42)
    assert np.array_equal(a, X.lic(T, 5.0, 1.0, 42))
    assert not np.array_equal(a, X.lic(T, 5.0, 1.0, 43))
    n = 64
    Tc = X.XformField.rotation(np.zeros((n, n)))
    norm = X.lic(Tc, 8.0, 1.2, 9, True)
    raw = X.lic(Tc, 8.0, 1.2, 9, False)
    assert orc.rel_l2(norm, raw) > 1e-6
    inner = np.zeros((n, n), bool)
    inner[8:n - 8, 8:n - 8] = True
    dev, cnt = _mean_deviation(orc, raw, 3.0, 0.0, 0.7, inner)
    assert cnt > 50
    assert dev < 5.0 * np.pi / 180


@pytest.mark.gpu
def test_cli_lic_matches_api(tmp_path):  # xconv_cli.cpp:602-639
    from paper_2006_13188_b200 import fileio as io
    n = 40
    ang = circular_field(n)
    fpath = str(tmp_path / "field.pfm")
    io.write_pfm_planes(fpath, [ang])
    out = str(tmp_path / "lic.pfm")
    r = subprocess.run([sys.executable, "-m", "paper_2006_13188_b200", "lic", "--field", fpath,
                        "--length", "5", "--line-width", "1", "--K", "12", "--seed", "3",
                        "--output", out], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = io.read_pfm_planes(out)[0]
    want = X.lic(X.XformField.rotation(io.read_xform(fpath, X.XformKind.rotation2).values),
                 5.0, 1.0, 3, True, 12)
    assert np.abs(got - want.astype(np.float32)).max() == 0.0
    import json
    side = json.load(open(out + ".json"))
    assert side["command"] == "lic" and side["parameters"]["seed"] == 3
    assert side["parameters"]["line-width"] == 1.0
