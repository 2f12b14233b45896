"""Images longer than the longest planned transform (4320) are cut into
halo-extended tiles (api.cu run_tiled): both pipelines read the signal and the
transformation field within R = ceil(r_max) of the output pixel only
(engine.hpp:300-319, 345-368), so every tile interior equals the full-image
result.  Checked against the spectral oracle at sampled pixels, with samples
on both sides of every tile seam and at the image corners (relative L2 <=
1e-5)."""
import ctypes as C

import numpy as np
import pytest

import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N

pytestmark = pytest.mark.gpu
TOL = 1e-5


def ofilter(orc, F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def _filter(r, R=9, m=4):
    from paper_2006_13188_b200 import workloads as WL
    return X.decompose_rotation2(WL.angular_filter(R, 3.5, m, r), R, R, 2 * m, 18, 20, float(R))


def _samples(r, h, w, R):
    ys = list(r.integers(0, h, 16)) + [0, h - 1, 0, h - 1]
    xs = list(r.integers(0, w, 16)) + [0, 0, w - 1, w - 1]
    for n, is_row in ((h, True), (w, False)):  # seams of the balanced split
        if n + R <= 4320:
            continue
        nt = -(-n // (4320 - 3 * R))
        t = -(-n // nt)
        for k in range(1, nt):
            for dlt in (-R - 1, -1, 0, R):
                p = min(max(k * t + dlt, 0), n - 1)
                q = int(r.integers(0, w if is_row else h))
                ys.append(p if is_row else q)
                xs.append(q if is_row else p)
    return np.asarray(ys), np.asarray(xs)


@pytest.mark.parametrize("h,w", [(4400, 260), (250, 4600), (8700, 200)])
@pytest.mark.parametrize("mode", [0, 1])
def test_tiled_matches_oracle(orc, h, w, mode):
    r = np.random.default_rng(h + w + mode)
    F = _filter(r)
    H = r.uniform(0, 1, (h, w)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
    fn = X.xcorr_fast if mode == 0 else X.xconv_fast
    res = fn(H, X.XformField.rotation(T), F)
    assert res.standard_ops == 9
    ys, xs = _samples(r, h, w, 9)
    ref = orc.spectral_oracle_at(mode, H, 0, T, ofilter(orc, F), ys, xs)
    assert orc.rel_l2(res.output[ys, xs], ref) < TOL


def test_tiled_colmajor_batch_f64_and_stats(orc):
    """The reference's layout (column-major), a batch with a shared field, fp64
    inputs and complex128 output; the stats report planned pads (no generic
    length) and every band."""
    r = np.random.default_rng(5)
    F = _filter(r)
    h, w, B = 4500, 180, 2
    H = r.uniform(0, 1, (B, h, w))
    T = r.uniform(0, 2 * np.pi, (h, w))
    Hc = np.ascontiguousarray(np.transpose(H, (0, 2, 1)))  # (B, w, h): y + x * h
    Tc = np.ascontiguousarray(T.T)
    out = np.zeros((B, w, h), np.complex128)
    ctx = N.context(0)
    d = N.ImageDesc(h, w, B, N.XC_F64, N.XC_F64, N.XC_C128, N.XC_COL_MAJOR, N.XC_HOST, 0, 0)
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), 0, C.byref(d), Hc.ctypes.data,
                           Tc.ctypes.data, None, 0, 0, out.ctypes.data, C.byref(st)), ctx.handle)
    assert st.standard_ops == 9 and max(st.pad_h, st.pad_w) <= 4320
    ys, xs = _samples(r, h, w, 9)
    for b in range(B):
        ref = orc.spectral_oracle_at(0, H[b].astype(np.float32), 0, T.astype(np.float32),
                                     ofilter(orc, F), ys, xs)
        # the oracle helper takes fp32 inputs: compare at the fp32 level
        got = out[b].T[ys, xs]
        assert orc.rel_l2(got, ref) < 1e-5 + 2e-6


def test_tiled_complex_signal_device_memory(orc):
    import torch
    r = np.random.default_rng(6)
    F = _filter(r)
    h, w = 300, 4400
    Hc = (r.uniform(0, 1, (h, w)) + 1j * r.uniform(-1, 1, (h, w))).astype(np.complex64)
    T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
    dev = torch.device("cuda", 0)
    dH, dT = torch.from_numpy(Hc).to(dev), torch.from_numpy(T).to(dev)
    dO = torch.zeros((h, w), dtype=torch.complex64, device=dev)
    torch.cuda.synchronize()
    ctx = N.context(0)
    d = N.ImageDesc(h, w, 1, N.XC_C64, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1, 0)
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), 1, C.byref(d), dH.data_ptr(),
                           dT.data_ptr(), None, 0, 0, dO.data_ptr(), C.byref(st)), ctx.handle)
    got = dO.cpu().numpy()
    # complex signal: real and imaginary parts scatter independently (linearity)
    ys, xs = _samples(r, h, w, 9)
    OF = ofilter(orc, F)
    ref = (orc.spectral_oracle_at(1, np.ascontiguousarray(Hc.real), 0, T, OF, ys, xs) +
           1j * orc.spectral_oracle_at(1, np.ascontiguousarray(Hc.imag), 0, T, OF, ys, xs))
    assert orc.rel_l2(got[ys, xs], ref) < TOL


@pytest.mark.parametrize("real_filter", [True, False])
def test_tiled_anglemax_matches_oracle(orc, real_filter):
    """xc_anglemax over tiles (api.cu anglemax_tiled): score and argmax at
    sampled pixels, seams included, against the oracle's angle max of the
    per-band responses (tensor-core path for the real filter, generic DFT
    kernel for the complex one)."""
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(11 + real_filter)
    R, m = 9, 4
    f = WL.angular_filter(R, 3.5, m, r)
    if real_filter:
        f = f.real + 0.0j
    F = X.decompose_rotation2(f, R, R, 2 * m, 18, 20, float(R))
    h, w = 4450, 150
    H = r.normal(0, 1, (h, w)).astype(np.float32)
    score, arg = X.anglemax(H, F, 360)
    ys, xs = _samples(r, h, w, R)
    Z = np.zeros((h, w), np.float32)
    G = np.stack([orc.spectral_oracle_at(0, H, 0, Z, orc.Filter(
        int(F.group), F.K, F.ks[i:i + 1], F.comps[:, i:i + 1], F.n_radii, F.n_angles, F.r_max,
        F.r_min, F.r_domain), ys, xs) for i in range(len(F.ks))])
    rs, ra = orc.anglemax(np.ascontiguousarray(G.reshape(len(F.ks), 1, -1)), F.ks, 360)
    assert orc.rel_l2(score[ys, xs], rs.ravel()) < TOL
    th = 2 * np.pi * np.arange(360) / 360
    S = np.abs(np.einsum("ka,kp->ap", np.exp(-1j * np.outer(th, np.asarray(F.ks)).T), G))
    top2 = np.sort(S, 0)[-2:]
    clear = (top2[1] - top2[0]) > 1e-4 * top2[1]
    assert clear.sum() >= len(ys) // 2
    assert np.array_equal(arg[ys, xs][clear], ra.ravel()[clear])
