"""Multi-rank sharding (world_size 2, gloo, CPU): band-sharded gather /
scatter / smoothing reduce to the single-process result.  The per-rank compute
is the CPU oracle here (the GPU path is the same orchestration with the
sm_100a compute and NCCL, exercised by bench.py --shard bands)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def oracle_compute(mode, H, T, F, components, inner_dc):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    OF = orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max, F.r_min,
                    F.r_domain)
    fn = orc.xcorr_fast if mode == 0 else orc.xconv_fast
    out = fn(np.asarray(H, np.complex128), int(T.kind), np.asarray(T.values, np.float64), OF,
             components=list(components))[0]
    if int(T.kind) == 1 and not inner_dc:  # remove the inner-DC term (engine.hpp:320-324)
        dc = orc.inner_dc_value(OF)
        out = out - (np.conj(dc) if mode == 0 else dc) * np.asarray(H, np.complex128)
    return out


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    import paper_2006_13188_b200 as X
    from paper_2006_13188_b200 import distributed as D
    res = {}
    rng = orc.Rng(300)
    n, R = 20, 5
    F = X.decompose_rotation2(rng.random_smooth_filter(R), R, R, 12, 16, 32, R)
    H = rng.random_field(n, n, True)
    T = X.XformField.rotation(rng.random_rotation_field(n, n))
    for mode in (0, 1):
        r = D.xfast_band_sharded(X.XMode(mode), H, T, F, compute=oracle_compute)
        if rank == 0:
            res[f"rot{mode}"] = (r.output, r.standard_ops)
    Fs = X.decompose_scale2(rng.annular_filter(R), R, R, 8, 48, 32, 1.0, R)
    S = X.XformField.scaling(rng.random_scale_field(n, n))
    for mode in (0, 1):
        r = D.xfast_band_sharded(X.XMode(mode), H, S, Fs, compute=oracle_compute)
        if rank == 0:
            res[f"scale{mode}"] = (r.output, r.standard_ops)
    sm = D.smooth_band_sharded(H.real.copy(), S, Fs, compute=oracle_compute)
    # bands k = +-1 only: the angular mean vanishes, so the filter integrates to
    # zero and every rank raises the reference's error (engine.hpp:388-392)
    i = [F.index_of(-1), F.index_of(1)]
    Z = X.FreqFilter2(0, F.K, [-1, 1], F.comps[:, i], F.n_radii, F.n_angles, F.r_max)
    try:
        D.smooth_band_sharded(H.real.copy(), T, Z, compute=oracle_compute)
        res["zero_integral"] = "no error"
    except ValueError as e:
        res["zero_integral"] = str(e)
    if rank == 0:
        res["smooth"] = (sm.output, sm.standard_ops, sm.clamped_pixels)
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_band_ranges_balanced():
    from paper_2006_13188_b200 import distributed as D
    assert [b - a for a, b in D.band_ranges(65, 8)] == [8, 8, 8, 8, 8, 8, 8, 9]
    assert sum(len(D.shard_components(range(-32, 33), r, 8)) for r in range(8)) == 65
    assert list(D.batch_range(16, 3, 8)) == [6, 7]


def test_band_sharded_world2_gloo(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = orc.Rng(300)
    n, R = 20, 5
    F = orc.decompose_rotation2(rng.random_smooth_filter(R), R, R, 12, 16, 32, R)
    H = rng.random_field(n, n, True)
    T = rng.random_rotation_field(n, n)
    for mode, fn in ((0, orc.xcorr_fast), (1, orc.xconv_fast)):
        out, ops = res[f"rot{mode}"]
        assert ops == 13 and orc.rel_l2(out, fn(H, 0, T, F)[0]) < 1e-12
    Fs = orc.decompose_scale2(rng.annular_filter(R), R, R, 8, 48, 32, 1.0, R)
    S = rng.random_scale_field(n, n)
    for mode, fn in ((0, orc.xcorr_fast), (1, orc.xconv_fast)):
        out, ops = res[f"scale{mode}"]
        assert ops == 9 and orc.rel_l2(out, fn(H, 1, S, Fs)[0]) < 1e-12
    out, ops, cl = res["smooth"]
    ref, rops, rcl = orc.smooth_adaptive(H.real.copy(), 1, S, Fs)
    assert ops == rops and cl == rcl and orc.rel_l2(out, ref) < 1e-12
    assert res["zero_integral"] == "normalization undefined: filter has zero integral"


def oracle_anglemax(H, F, n_angles, components):
    """Per-rank angle max on the CPU oracle: G_k = H (*) F_k (theta = 0 keeps the
    band response unsteered), then the per-pixel max over n_angles rotations."""
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    OF = orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max, F.r_min,
                    F.r_domain)
    ks = list(components) if components else [int(k) for k in F.ks]
    Hc = np.asarray(H, np.complex128)
    zero = np.zeros(Hc.shape)
    G = np.stack([orc.xcorr_fast(Hc, 0, zero, OF, components=[k])[0] for k in ks])
    return orc.anglemax(G, ks, n_angles)


def _match_case(orc):
    """A small matching problem: noise with two rotated copies of a template."""
    rng = np.random.default_rng(5)
    h, w, R = 37, 30, 4
    tpl = rng.normal(size=(2 * R + 1, 2 * R + 1))
    img = rng.normal(size=(h, w)) * 0.3
    for (y, x) in ((9, 8), (27, 20)):
        img[y - R:y + R + 1, x - R:x + R + 1] += np.rot90(tpl, (y + x) % 4)
    F = orc.decompose_rotation2(tpl + 0j, R, R, 8, 8, 24, R)
    return img, F


def _spatial_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    import paper_2006_13188_b200 as X
    from paper_2006_13188_b200 import distributed as D
    img, OF = _match_case(orc)
    R = 4
    F = X.FreqFilter2(0, OF.K, OF.ks, OF.comps, OF.n_radii, OF.n_angles, OF.r_max)
    sa = D.anglemax_spatial_sharded(img, F, 36, compute=oracle_anglemax)
    pk = D.match_peaks_spatial_sharded(img, F, 3.0, 0.5, 36, compute=oracle_anglemax)
    pk2 = D.match_peaks_spatial_sharded(img, F, 6.5, 0.2, 36, components=[-2, 0, 2],
                                        compute=oracle_anglemax)
    if rank == 0:
        q.put({"score": sa[0], "arg": sa[1], "peaks": [(p.x, p.y, p.value) for p in pk],
               "peaks2": [(p.x, p.y, p.value) for p in pk2], "R": R})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_spatial_sharded_anglemax_and_peaks_gloo(orc, world):
    """Row-strip sharding of the angle max (SURVEY 8(e) caveat 3): the gathered
    score/argmax equal the whole-image oracle, and the merged peaks equal the
    whole-image find_peaks exactly (positions, order) with values to 1e-12."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spatial_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    img, OF = _match_case(orc)

    score, arg = oracle_anglemax(img, OF, 36, None)
    assert orc.rel_l2(res["score"], score) < 1e-12
    assert np.array_equal(res["arg"], arg)
    for key, radius, frac, comp in (("peaks", 3.0, 0.5, None), ("peaks2", 6.5, 0.2, [-2, 0, 2])):
        s = score if comp is None else oracle_anglemax(img, OF, 36, comp)[0]
        ref = orc.find_peaks(s, radius, frac)
        got = res[key]
        assert len(got) == len(ref) >= 2
        assert [(x, y) for x, y, _ in got] == [(x, y) for x, y, _ in ref]
        assert np.allclose([v for _, _, v in got], [v for _, _, v in ref], rtol=1e-12, atol=0)


# ------------------------------------------------- pair-aware band sharding

def test_shard_components_in_pairs_covers_and_stays_symmetric():
    """Real signals run +-k pairs (only k >= 0 is transformed), so every rank's
    share must be symmetric, the shares disjoint, and the loads (bands k >= 0)
    balanced to +-1 (api.cu shard_bands / shard_in_pairs)."""
    from paper_2006_13188_b200 import distributed as D
    ks = list(range(-32, 33))
    for world in (1, 2, 3, 4, 8):
        shares = [D.shard_components(ks, r, world, pairs=True) for r in range(world)]
        assert sorted(k for s in shares for k in s) == ks
        loads = []
        for s in shares:
            assert all(-k in s for k in s)
            loads.append(sum(1 for k in s if k >= 0))
        assert max(loads) - min(loads) <= 1
    # more ranks than non-negative bands: the extra ranks get nothing
    shares = [D.shard_components([-1, 0, 1], r, 4, pairs=True) for r in range(4)]
    assert sorted(k for s in shares for k in s) == [-1, 0, 1]
    # contiguous ranges by default
    assert D.shard_components(ks, 0, 8) == list(range(-32, -24))


def test_shard_in_pairs_rule():
    import paper_2006_13188_b200 as X
    from paper_2006_13188_b200 import distributed as D
    from paper_2006_13188_b200.engine import XMode
    ks = np.arange(-2, 3)
    r = np.random.default_rng(3)
    comps = r.normal(size=(6, 5)) + 1j * r.normal(size=(6, 5))
    F = X.FreqFilter2(0, 4, ks, comps, 6, 16, 5.0)
    assert not F.hermitian()
    herm = comps.copy()
    herm[:, 0], herm[:, 1], herm[:, 2] = np.conj(comps[:, 4]), np.conj(comps[:, 3]), comps[:, 2].real
    FH = X.FreqFilter2(0, 4, ks, herm, 6, 16, 5.0)
    assert FH.hermitian()
    real, cplx = np.zeros((4, 4), np.float32), np.zeros((4, 4), np.complex64)
    assert D.shard_in_pairs(XMode.convolution, real, F, ks)       # conjugate band pairs
    assert not D.shard_in_pairs(XMode.correlation, real, F, ks)   # gather needs F_-k = conj F_k
    assert D.shard_in_pairs(XMode.correlation, real, FH, ks)      # Hermitian half-band
    assert not D.shard_in_pairs(XMode.convolution, cplx, F, ks)   # complex signal
    assert not D.shard_in_pairs(XMode.convolution, real, F, [2, 1, 0, -1])  # asymmetric
