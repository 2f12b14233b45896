"""3D parts of the file formats and CLI (SURVEY 8(f) F3 with F4): the XCF1
container for SphFilter3 (io.hpp:318-368), `decompose --group rotation3d`
(xconv_cli.cpp:739-780) and `steer3d` (xconv_cli.cpp:191-204, 645-688).  Host
work only, so these run on CPU; the oracle checks the steering."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import fileio as io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _filter3(orc, R=3, K=3):
    vol = np.real(orc.Rng(93).random_smooth_filter3(R))
    return vol, X.decompose_rotation3(vol, R, R, R, K, 2 * R, float(R), 12, 12)


def test_filter3_container_round_trip_and_layout(orc, tmp_path):
    _, F = _filter3(orc)
    p = str(tmp_path / "f3.xcf")
    io.write_filter3(p, F)
    data = open(p, "rb").read()
    assert data[:4] == b"XCF1" and data[4] == 2
    K, nr, zero = struct.unpack_from("<iii", data, 5)
    assert (K, nr, zero) == (F.K, F.n_radii, 0)
    rows, cols = struct.unpack_from("<qq", data, 5 + 12 + 24)
    assert (rows, cols) == F.coeffs.shape and cols == (F.K + 1) ** 2
    G = io.read_filter3(p)
    assert G.K == F.K and G.n_radii == F.n_radii and G.r_max == F.r_max
    assert np.array_equal(G.coeffs, F.coeffs)
    with pytest.raises(io.IoError, match="not a 3D filter"):
        F2 = X.decompose_rotation2(np.ones((9, 9)), 4, 4, 4, 8, 16, 4.0)
        q = str(tmp_path / "f2.xcf")
        io.write_filter(q, F2)
        io.read_filter3(q)
    open(p, "wb").write(data[:-8])
    with pytest.raises(io.IoError, match="truncated"):
        io.read_filter3(p)


def test_steer_filter3_matches_reference_mixing(orc):
    _, F = _filter3(orc)
    q = orc.Rng(5).random_quaternion()
    G = X.steer_filter3(F, q)
    # xconv_cli.cpp:191-204, element by element with the oracle's Wigner D
    for l in range(F.K + 1):
        D = orc.wigner_d(l, q)
        for j in range(F.n_radii):
            c = np.array([F.coeff(j, l, m) for m in range(-l, l + 1)])
            want = D @ c
            got = np.array([G.coeff(j, l, m) for m in range(-l, l + 1)])
            assert np.abs(got - want).max() < 1e-12
    # identity leaves the filter unchanged; q then q^-1 restores it
    assert np.abs(X.steer_filter3(F, [1, 0, 0, 0]).coeffs - F.coeffs).max() < 1e-12
    qi = np.array([q[0], -q[1], -q[2], -q[3]])
    assert np.abs(X.steer_filter3(G, qi).coeffs - F.coeffs).max() < 1e-10


def test_cli_decompose3_and_steer3d(orc, tmp_path):
    vol, _ = _filter3(orc)
    stack = str(tmp_path / "vol.pfm")
    io.write_pfm_planes(stack, [vol[z] for z in range(vol.shape[0])])
    f3 = str(tmp_path / "f3.xcf")
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2006_13188_b200", *a],
                                    cwd=ROOT, capture_output=True, text=True)
    r = run("decompose", "--input", stack, "--group", "rotation3d", "--K", "3", "--output", f3)
    assert r.returncode == 0, r.stderr
    F = io.read_filter3(f3)
    n = vol.shape[0]
    R = (n - 1) / 2.0
    want = X.decompose_rotation3(vol.astype(np.float32).astype(np.float64), R, R, R, 3,
                                 2 * int(np.ceil(R)), R)
    assert np.abs(F.coeffs - want.coeffs).max() < 1e-12
    side = json.load(open(f3 + ".json"))
    assert side["counters"]["steering-products"] == 1 + 9 + 25 + 49
    out = str(tmp_path / "rot.pfm")
    q = [0.9, 0.1, -0.3, 0.2]
    r = run("steer3d", "--filter", f3, "--quat", *map(str, q), "--output", out)
    assert r.returncode == 0, r.stderr
    planes = io.read_pfm_planes(out)
    Rr = int(np.ceil(F.r_max))
    assert len(planes) == 2 * Rr + 1 and planes[0].shape == (2 * Rr + 1, 2 * Rr + 1)
    qn = np.array(q) / np.linalg.norm(q)
    ref = X.reconstruct3(X.steer_filter3(F, qn), 2 * Rr + 1, 2 * Rr + 1, 2 * Rr + 1,
                         Rr, Rr, Rr)
    assert np.abs(np.stack(planes) - ref.real.astype(np.float32)).max() == 0.0
    assert run("steer3d", "--filter", f3, "--quat", "0", "0", "0", "0",
               "--output", out).returncode == 2
