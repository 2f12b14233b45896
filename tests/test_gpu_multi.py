"""Multi-GPU contexts of the C ABI (include/xconv_b200.h
xc_context_create_multi / xc_context_create_rank): xc_run / xc_smooth split
the bands (engine.hpp:300-319, 345-368) over the context's devices and sum
the partials inside the library.

The pool has one GPU, so:
  * Context.multi([0]) and Context.rank(0, id, 0, 1) run the NCCL plumbing
    (communicator init, ncclReduce) with one device;
  * Context.multi([0, 0, 0]) lists device 0 three times: three child contexts
    each run a band range (the scale inner-DC term on the first only) and the
    peer-copy reduce sums them in device order -- the orchestration of an
    8-GPU run, checked against the oracle and the single-device result.
"""
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


def _rot_case(orc, seed=91, n=40, R=6, K=12):
    rng = orc.Rng(seed)
    F = X.decompose_rotation2(rng.random_smooth_filter(R), R, R, K, 16, 32, R)
    H = rng.random_field(n, n, True)
    T = rng.random_rotation_field(n, n)
    return F, H, T


def _scale_case(orc, seed=92, n=36, R=6):
    rng = orc.Rng(seed)
    F = X.decompose_scale2(rng.annular_filter(R), R, R, 8, 48, 32, 1.0, R)
    H = rng.random_field(n, n, False)
    S = rng.random_scale_field(n, n)
    return F, H, S


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("mode", [0, 1])
def test_multi_rotation_bands(orc, devices, mode):
    F, H, T = _rot_case(orc)
    ctx = N.Context.multi(devices)
    assert ctx.devices() == (len(devices), len(devices) == 1)
    fn = X.xcorr_fast if mode == 0 else X.xconv_fast
    r = fn(H, X.XformField.rotation(T), F, ctx=ctx)
    one = fn(H, X.XformField.rotation(T), F)
    ref = (orc.xcorr_fast if mode == 0 else orc.xconv_fast)(H, 0, T, ofilter(orc, F))[0]
    assert r.standard_ops == one.standard_ops == F.n_components()
    assert orc.rel_l2(r.output, ref) < TOL
    if len(devices) == 1:
        assert np.array_equal(r.output, one.output)  # one device: the same kernels
    else:
        assert orc.rel_l2(r.output, one.output) < 1e-6


@pytest.mark.parametrize("mode", [0, 1])
def test_multi_scale_inner_dc_once(orc, mode):
    F, H, S = _scale_case(orc)
    ctx = N.Context.multi([0, 0, 0])
    fn = X.xcorr_fast if mode == 0 else X.xconv_fast
    r = fn(H, X.XformField.scaling(S), F, ctx=ctx)
    ref = (orc.xcorr_fast if mode == 0 else orc.xconv_fast)(H, 1, S, ofilter(orc, F))[0]
    assert orc.rel_l2(r.output, ref) < TOL


def test_multi_band_subset_and_more_devices_than_bands(orc):
    F, H, T = _rot_case(orc)
    ctx = N.Context.multi([0] * 5)
    plan = X.XConvPlan(components=[-2, 0, 3])  # 3 bands over 5 devices: 2 add zeros
    r = X.xcorr_fast(H, X.XformField.rotation(T), F, plan, ctx=ctx)
    ref = orc.xcorr_fast(H, 0, T, ofilter(orc, F), components=[-2, 0, 3])[0]
    assert r.standard_ops == 3
    assert orc.rel_l2(r.output, ref) < TOL
    with pytest.raises(ValueError, match="plan retains a component the filter lacks"):
        X.xcorr_fast(H, X.XformField.rotation(T), F, X.XConvPlan(components=[99]), ctx=ctx)


@pytest.mark.parametrize("devices", [[0], [0, 0, 0]])
def test_multi_smoothing(orc, devices):
    F, H, S = _scale_case(orc)
    ctx = N.Context.multi(devices)
    got = X.smooth_adaptive(H.real.copy(), X.XformField.scaling(S), F, device=ctx)
    ref, ops, clamped = orc.smooth_adaptive(H.real.copy(), 1, S, ofilter(orc, F))
    assert got.standard_ops == ops and got.clamped_pixels == clamped
    assert orc.rel_l2(got.output, ref) < TOL


def test_multi_guard_error_and_zero_integral(orc):
    F, H, S = _scale_case(orc)
    ctx = N.Context.multi([0, 0])
    bad = S.copy()
    bad[3, 5] = 1e6  # y = 3, x = 5 (test_engine_scale.cpp:161-178)
    with pytest.raises(ValueError, match=r"guard band.*|\(5,3\)") as e:
        X.xcorr_fast(H, X.XformField.scaling(bad), F, ctx=ctx)
    assert "(5,3)" in str(e.value) and "guard band" in str(e.value)
    Fr, Hr, T = _rot_case(orc)
    i = [Fr.index_of(-1), Fr.index_of(1)]
    Z = X.FreqFilter2(0, Fr.K, [-1, 1], Fr.comps[:, i], Fr.n_radii, Fr.n_angles, Fr.r_max)
    with pytest.raises(ValueError, match="normalization undefined: filter has zero integral"):
        X.smooth_adaptive(Hr.real.copy(), X.XformField.rotation(T), Z, device=ctx)


def test_multi_batch_sharding(orc):
    F, _, _ = _rot_case(orc)
    r = np.random.default_rng(4)
    H = r.random((5, 32, 40)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (5, 32, 40)).astype(np.float32)
    ctx = N.Context.multi([0, 0], shard=N.XC_SHARD_BATCH)
    got = X.xcorr_fast(H, X.XformField.rotation(T), F, ctx=ctx).output
    one = X.xcorr_fast(H, X.XformField.rotation(T), F).output
    assert np.array_equal(got, one)
    Fs, _, _ = _scale_case(orc)
    S = np.exp(r.uniform(np.log(0.5), np.log(2.0), (5, 32, 40))).astype(np.float32)
    sm = X.smooth_adaptive(H, X.XformField.scaling(S), Fs, device=ctx)
    sm1 = X.smooth_adaptive(H, X.XformField.scaling(S), Fs)
    assert np.array_equal(sm.output, sm1.output) and sm.clamped_pixels == sm1.clamped_pixels


def test_multi_device_memory_and_accumulate(orc):
    import torch
    F, H, T = _rot_case(orc)
    ctx = N.Context.multi([0, 0, 0])
    n = H.shape[0]
    hs = torch.from_numpy(H.astype(np.complex64)).cuda()
    ts = torch.from_numpy(T.astype(np.float32)).cuda()
    out = torch.ones((n, n), dtype=torch.complex64, device="cuda")
    d = N.ImageDesc(n, n, 1, N.XC_C64, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1,
                    N.XC_ROTATION2)
    st = N.Stats()
    N.check(N.lib().xc_run(ctx.handle, F.handle(), 0, C.byref(d), C.c_void_p(hs.data_ptr()),
                           C.c_void_p(ts.data_ptr()), None, 0, N.XC_FLAG_ACCUMULATE,
                           C.c_void_p(out.data_ptr()), C.byref(st)), ctx.handle)
    torch.cuda.synchronize()
    ref = orc.xcorr_fast(H, 0, T, ofilter(orc, F))[0]
    assert st.standard_ops == F.n_components()
    assert orc.rel_l2(out.cpu().numpy() - 1.0, ref) < TOL


def test_rank_context_single_rank_nccl(orc):
    F, H, T = _rot_case(orc)
    ctx = N.Context.rank(0, N.nccl_unique_id(), 0, 1)
    assert ctx.devices() == (1, True)
    r = X.xcorr_fast(H, X.XformField.rotation(T), F, ctx=ctx)
    one = X.xcorr_fast(H, X.XformField.rotation(T), F)
    assert np.array_equal(r.output, one.output)
    Fs, Hs, S = _scale_case(orc)
    sm = X.smooth_adaptive(Hs.real.copy(), X.XformField.scaling(S), Fs, device=ctx)
    ref = orc.smooth_adaptive(Hs.real.copy(), 1, S, ofilter(orc, Fs))[0]
    assert orc.rel_l2(sm.output, ref) < TOL


def test_rank_context_async_reduce(orc):
    """XC_FLAG_ASYNC: the reduce of call i is queued on the context's comm
    stream and overlaps call i + 1 (two partial slots); after
    xc_context_synchronize both outputs equal the synchronous result."""
    import torch
    F, H, T = _rot_case(orc)
    n = H.shape[0]
    ctx = N.Context.rank(0, N.nccl_unique_id(), 0, 1)
    hs = torch.from_numpy(H.astype(np.complex64)).cuda()
    ts = torch.from_numpy(T.astype(np.float32)).cuda()
    outs = [torch.zeros((n, n), dtype=torch.complex64, device="cuda") for _ in range(3)]
    d = N.ImageDesc(n, n, 1, N.XC_C64, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1,
                    N.XC_ROTATION2)
    st = N.Stats()
    for o in outs:
        N.check(N.lib().xc_run(ctx.handle, F.handle(), 0, C.byref(d), C.c_void_p(hs.data_ptr()),
                               C.c_void_p(ts.data_ptr()), None, 0, N.XC_FLAG_ASYNC,
                               C.c_void_p(o.data_ptr()), C.byref(st)), ctx.handle)
    ctx.synchronize()
    one = X.xcorr_fast(H.astype(np.complex64), X.XformField.rotation(T.astype(np.float32)), F)
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), one.output)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0]])
@pytest.mark.parametrize("real_filter", [False, True])
def test_multi_pair_sharding_real_signal(orc, devices, real_filter):
    """A real signal at a pair-plan pad (1152): the bands are shared out in +-k
    pairs (api.cu shard_in_pairs), so every device keeps the conjugate-pair
    (scatter) or Hermitian half-band (real filter, gather and scatter) mode and
    transforms its bands k >= 0 only; the summed result matches the oracle."""
    from paper_2006_13188_b200 import workloads as WL
    r = np.random.default_rng(77)
    f = WL.angular_filter(10, 4.0, 5, r)
    if real_filter:
        f = f.real + 0.0j
    F = X.decompose_rotation2(f, 10, 10, 10, 20, 24, 10.0)
    n = 1030
    H = r.uniform(0, 1, (n, n)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (n, n)).astype(np.float32)
    ctx = N.Context.multi(devices)
    ys, xs = r.integers(0, n, 48), r.integers(0, n, 48)
    for mode, fn in ((1, X.xconv_fast), (0, X.xcorr_fast)):
        res = fn(H, X.XformField.rotation(T), F, ctx=ctx)
        ref = orc.spectral_oracle_at(mode, H, 0, T, ofilter(orc, F), ys, xs)
        assert res.standard_ops == 11
        assert orc.rel_l2(res.output[ys, xs], ref) < TOL


_PEER_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2006_13188_b200 as X
from paper_2006_13188_b200 import _native as N
r = np.random.default_rng(5)
from paper_2006_13188_b200 import workloads as WL
F = X.decompose_rotation2(WL.angular_filter(6, 2.5, 4, r), 6, 6, 8, 12, 20, 6.0)
H = r.uniform(0, 1, (2, 70, 90)).astype(np.float32)
T = r.uniform(0, 6.28, (2, 70, 90)).astype(np.float32)
ctx = N.Context.multi([0, 0, 0])
a = X.xcorr_fast(H, X.XformField.rotation(T), F, ctx=ctx).output
b = X.xconv_fast(H, X.XformField.rotation(T), F, ctx=ctx).output
FS = X.decompose_scale2(np.exp(-((np.mgrid[-6:7, -6:7] ** 2).sum(0)) / 18.0) + 0j, 6, 6, 6, 32, 24, 1.0, 6)
S = np.exp(r.uniform(0, 0.4, (70, 90))).astype(np.float32)
c = X.smooth_adaptive(H[0], X.XformField.scaling(S), FS, device=ctx).output
np.savez(sys.argv[2], a=a, b=b, c=c)
"""


def test_peer_write_partials_equal_the_copy_reduce(tmp_path):
    """Multi-device contexts write every device's partial straight into the
    root's memory (api.cu peer_slots) and add the slots in device order; with
    XCB_PEER_WRITE=0 the partials stay local and go through the reduce.  Both
    add in the same order, so the outputs are bit-identical (gather, scatter,
    smoothing; batches)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        f = tmp_path / f"pw{flag}.npz"
        env = dict(os.environ, XCB_PEER_WRITE=flag)
        subprocess.run([sys.executable, "-c", _PEER_SCRIPT, root, str(f)], check=True, env=env,
                       timeout=600)
        outs.append(np.load(f))
    for k in ("a", "b", "c"):
        assert np.isfinite(outs[0][k]).all()
        assert np.array_equal(outs[0][k], outs[1][k]), k
