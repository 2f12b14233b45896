"""GPU parity at every pair-plan transform length (k_pair.cu XCB_PAIR_TABLE).
The pad rule (api.cu pick_pad2d) sends most image sizes to one of these
lengths, so each gets a gather (xcorr_fast), a scatter (xconv_fast: conjugate
band pairs where S2 fits, complex signal on the full path) and an angle max
case, each against the spectral oracle at sampled pixels (relative L2 <= 1e-5,
fp32 GPU vs the double oracle; exact argmax at the sampled pixels).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N

pytestmark = pytest.mark.gpu
TOL = 1e-5
LENGTHS = [288, 576, 768, 1024, 1152, 1280, 1536, 1920, 2048, 2160, 2304, 2560, 2880, 3072, 3456,
           4096, 4320]


def ofilter(orc, F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def _case(L, seed):
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(seed + L)
    R, m = 9, 4
    F = X.decompose_rotation2(WL.angular_filter(R, 3.5, m, r), R, R, 2 * m, 18, 20, float(R))
    n = L - R - 2 - int(r.integers(0, 20))  # pad rule: the least length >= n + R
    w = max(64, n // 3 + int(r.integers(0, 7)))  # a short second axis keeps the oracle cheap
    return r, F, n, w


def _pads(F, h, w, mode):
    ctx = N.context(0)
    H = np.zeros((h, w), np.float32)
    out = np.zeros((h, w), np.complex64)
    d = N.ImageDesc(h, w, 1, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_HOST, 1, 0)
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), mode, C.byref(d), H.ctypes.data,
                           H.ctypes.data, None, 0, 0, out.ctypes.data, C.byref(st)), ctx.handle)
    return st.pad_h, st.pad_w


@pytest.mark.parametrize("L", LENGTHS)
@pytest.mark.parametrize("axis", ["rows", "cols"])
def test_pair_length_gather_and_scatter(orc, L, axis):
    r, F, n, w = _case(L, 0 if axis == "rows" else 1000)
    h, wd = (w, n) if axis == "rows" else (n, w)  # row transforms have length Pw
    H = r.uniform(0, 1, (h, wd)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (h, wd)).astype(np.float32)
    ph, pw = _pads(F, h, wd, 0)
    assert (pw if axis == "rows" else ph) == L
    ys = np.concatenate([r.integers(0, h, 24), [0, h - 1, 0, h - 1]])
    xs = np.concatenate([r.integers(0, wd, 24), [0, 0, wd - 1, wd - 1]])
    OF = ofilter(orc, F)
    for mode, fn in ((0, X.xcorr_fast), (1, X.xconv_fast)):
        got = fn(H, X.XformField.rotation(T), F).output
        ref = orc.spectral_oracle_at(mode, H, 0, T, OF, ys, xs)
        assert orc.rel_l2(got[ys, xs], ref) < TOL, (mode, L)


@pytest.mark.parametrize("L", [576, 1024, 1536, 2048, 2880, 4096])
def test_pair_length_complex_scatter_and_anglemax(orc, L):
    """A complex signal (full scatter path, no band pairing) and the angle max
    planes at a selection of the new lengths (square pads)."""
    r, F, n, _ = _case(L, 2000)
    h = w = n
    ys, xs = r.integers(0, h, 16), r.integers(0, w, 16)
    OF = ofilter(orc, F)
    if L <= 2048:  # the complex oracle below is a full-image fp64 run
        Hc = (r.uniform(0, 1, (h, w)) + 1j * r.uniform(-1, 1, (h, w))).astype(np.complex64)
        T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
        got = X.xconv_fast(Hc, X.XformField.rotation(T), F).output
        ref = orc.xconv_fast(Hc.astype(np.complex128), 0, T.astype(np.float64), OF,
                             nthreads=16)[0]
        assert orc.rel_l2(got[ys, xs], ref[ys, xs]) < TOL
    H = r.normal(0, 1, (h, w)).astype(np.float32)
    score, arg = X.anglemax(H, F, 360)
    # per-band responses G_k = H (*) F_k at the pixels: the gather with theta = 0
    # and a one-band filter; then the oracle's own angle max over those columns
    Z = np.zeros((h, w), np.float32)
    G = np.stack([orc.spectral_oracle_at(0, H, 0, Z, orc.Filter(
        int(F.group), F.K, F.ks[i:i + 1], F.comps[:, i:i + 1], F.n_radii, F.n_angles, F.r_max,
        F.r_min, F.r_domain), ys, xs) for i in range(len(F.ks))])
    rs, ra = orc.anglemax(np.ascontiguousarray(G.reshape(len(F.ks), 1, -1)), F.ks, 360)
    assert orc.rel_l2(score[ys, xs], rs.ravel()) < TOL
    # exact argmax where the maximum is separated from the runner-up by > 1e-4 relative
    th = 2 * np.pi * np.arange(360) / 360
    S = np.abs(np.einsum("ka,kp->ap", np.exp(-1j * np.outer(th, np.asarray(F.ks)).T), G))
    top2 = np.sort(S, 0)[-2:]
    clear = (top2[1] - top2[0]) > 1e-4 * top2[1]
    assert clear.sum() >= len(ys) // 2
    assert np.array_equal(arg[ys, xs][clear], ra.ravel()[clear])
