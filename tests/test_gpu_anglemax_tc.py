"""The tensor-core angle max (csrc/k_anglemax_tc.cu: E/O parity split, two
tf32 GEMMs per 128-pixel tile, 3xTF32, tcgen05.mma into TMEM) against the
oracle's 360-angle maximum of the band responses (score at relative L2
<= 1e-5; the angle it picks attains the oracle's maximum to 1e-5) and against
the CUDA-core kernel (XCB_ANGLE_TC=0, another process).  Real templates with
band limits |m| <= 4, 8, 16 (KH = 4, 8, 16), image sizes whose pixel count is
not a multiple of the 128-pixel tile, a batch, f64 scores.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2006_13188_b200 as X

pytestmark = pytest.mark.gpu
TOL = 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ofilter(orc, F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def _case(orc, K, h, w, seed):
    rng = np.random.default_rng(seed)
    R = 9
    y, x = np.mgrid[-R:R + 1, -R:R + 1].astype(np.float64)
    tpl = np.zeros_like(x)
    for _ in range(4):
        cx, cy, s, a = rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(1, 2.5), rng.normal()
        tpl += a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * s * s))
    tpl *= np.exp(-(x * x + y * y) / (2 * (0.45 * R) ** 2))
    F = X.decompose_rotation2(tpl, R, R, K, 2 * R, 2 * K + 2, R + 0.5)
    H = rng.standard_normal((h, w)).astype(np.float32)
    return F, H


def _oracle(orc, H, F):
    OF = ofilter(orc, F)
    Hd = H.astype(np.float64)
    G = np.stack([orc.xcorr_fast(Hd, 0, np.zeros_like(Hd), OF, components=[int(k)])[0]
                  for k in OF.ks])
    return G, OF.ks, orc.anglemax(G, OF.ks, 360)


def _attains(G, ks, arg, oscore):
    at = np.abs(np.einsum("kyx,kyx->yx", G,
                          np.exp(-2j * np.pi * np.asarray(ks)[:, None, None] * arg[None] / 360)))
    return np.all(at >= oscore * (1 - TOL) - 1e-9)


@pytest.mark.parametrize("K,h,w", [(8, 61, 97), (16, 128, 130), (32, 75, 203), (32, 1, 1)])
def test_tc_anglemax_matches_oracle(orc, K, h, w):
    F, H = _case(orc, K, h, w, K + h)
    score, arg = X.anglemax(H, F, 360)
    G, ks, (oscore, oarg) = _oracle(orc, H, F)
    assert orc.rel_l2(score, oscore) < TOL, orc.rel_l2(score, oscore)
    assert _attains(G, ks, arg, oscore)
    if h * w > 1:  # (one pixel: G_0 only, all 360 angles tie up to rounding)
        assert np.mean(arg == oarg) > 0.999  # near-ties aside, the same (first) angle


def test_tc_anglemax_batch_and_f64(orc):
    F, H = _case(orc, 32, 90, 110, 5)
    B = np.stack([H, 0.5 * H[::-1].copy(), np.zeros_like(H)]).astype(np.float64)
    score, arg = X.anglemax(B, F, 360)
    assert score.dtype == np.float64
    for i in range(2):
        G, ks, (oscore, _) = _oracle(orc, B[i].astype(np.float32), F)
        assert orc.rel_l2(score[i], oscore) < TOL
    assert np.all(score[2] == 0)


def test_tc_matches_cuda_core_kernel(tmp_path):
    from paper_2006_13188_b200 import workloads as WL  # noqa: F401
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2006_13188_b200 as X\n"
            "from paper_2006_13188_b200 import workloads as WL\n"
            "w = WL.config3(n=1024, n_templates=2)\n"
            "s, a = X.anglemax(w.signal[0], w.filt, 360)\n"
            "np.savez(sys.argv[1], s=s, a=a)\n") % ROOT
    out = {}
    for flag in ("1", "0"):
        p = str(tmp_path / f"am{flag}.npz")
        subprocess.run([sys.executable, "-c", code, p], check=True, timeout=600,
                       env=dict(os.environ, XCB_ANGLE_TC=flag))
        out[flag] = np.load(p)
    s1, s0 = out["1"]["s"], out["0"]["s"]
    assert np.linalg.norm(s1 - s0) / np.linalg.norm(s0) < 2e-6
    assert np.mean(out["1"]["a"] == out["0"]["a"]) > 0.999
