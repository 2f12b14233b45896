"""Committed 3D golden fixtures (tests/golden/3d/*.npz, made by
make_golden3d.py from the 3D oracle on the reference's seeded fixtures): the
oracle must keep reproducing them and the host decomposition must match them
(CPU); xcorr_fast_3d / xconv_fast_3d must match them on the GPU (rel L2
<= 1e-5)."""
import glob
import os

import numpy as np
import pytest

import paper_2006_13188_b200 as X

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "3d")
FILES = sorted(glob.glob(os.path.join(HERE, "*.npz")))
IDS = [os.path.basename(f) for f in FILES]


def load(path):
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("path", FILES, ids=IDS)
def test_oracle_and_host_decomposition_reproduce_golden3d(orc, path):
    d = load(path)
    R, K, ns = int(d["R"]), int(d["K"]), int(d["ns"])
    F = orc.decompose_rotation3(d["vol"], R, R, R, K, 2 * R, float(R), ns, ns)
    assert np.abs(F.coeffs - d["coeffs"]).max() < 1e-13
    G = X.decompose_rotation3(d["vol"], R, R, R, K, 2 * R, float(R), ns, ns)
    assert np.abs(G.coeffs - d["coeffs"]).max() < 1e-12 * np.abs(d["coeffs"]).max()
    out, ops = orc.xfast3(0, d["signal"], d["quats"], F)
    assert ops == int(d["ops"]) and orc.rel_l2(out, d["xcorr"]) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("path", FILES, ids=IDS)
def test_gpu_matches_golden3d(orc, path):
    d = load(path)
    R, K = int(d["R"]), int(d["K"])
    F = X.SphFilter3(K, 2 * R, float(R), d["coeffs"])
    T = X.rotation3d(d["quats"])
    H = d["signal"] if np.any(d["signal"].imag) else d["signal"].real
    r = X.xcorr_fast_3d(H, T, F)
    assert r.standard_ops == int(d["ops"])
    assert orc.rel_l2(r.output, d["xcorr"]) < 1e-5
    assert orc.rel_l2(X.xconv_fast_3d(H, T, F).output, d["xconv"]) < 1e-5
