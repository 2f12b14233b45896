"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed).

SURVEY 8(e): the bands are independent terms of the extended sum
(engine.hpp:300-319, 345-368) and XConvPlan::components (engine.hpp:19)
already expresses a band subset, so

  * band sharding: rank g runs xcorr_fast / xconv_fast on a contiguous band
    range (balanced to +-1) and the partial outputs are summed with one
    reduce (NCCL over NVLink on GPUs, gloo in the CPU tests).  The scale
    group's inner-DC term (engine.hpp:320-324 / 369-371) is added by the root
    rank only (XC_FLAG_NO_INNER_DC elsewhere).  smooth_adaptive is nonlinear:
    numerator and denominator are reduced separately and divided on the root
    with the reference's 1e-9 floor (engine.hpp:405-418).
  * batch sharding: images are split across ranks, no collective at all.

The per-rank compute is injectable (`compute(mode, H, T, F, components,
inner_dc)`) so the orchestration is testable on CPU; the default is the
product's own GPU path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .engine import (FreqFilter2, Response2, SmoothResult, XConvPlan, XformField, XformKind,
                     XMode, _fast)


def band_ranges(n: int, world: int):
    """Contiguous ranges balanced to +-1 (65 bands over 8 ranks: 9,8,...,8)."""
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


def shard_components(ks, rank: int, world: int, pairs: bool = False) -> list:
    """This rank's bands: a contiguous range of `ks`, or (pairs, see
    shard_in_pairs) a contiguous range of the bands k >= 0 with their -k
    partners, so that the share stays symmetric."""
    ks = [int(k) for k in ks]
    if not pairs:
        a, b = band_ranges(len(ks), world)[rank]
        return ks[a:b]
    nn = [k for k in ks if k >= 0]
    a, b = band_ranges(len(nn), world)[rank]
    mine = set(nn[a:b])
    return [k for k in ks if abs(k) in mine]


def shard_in_pairs(mode, H, F, ks) -> bool:
    """Mirror of the library's rule (api.cu shard_in_pairs): a real signal with a
    symmetric band selection runs in +-k pairs, transforming the bands k >= 0
    only (Hermitian half-band mode for a real filter, the scatter's conjugate
    band pairs for any filter), so shares must hold whole pairs."""
    if np.iscomplexobj(np.asarray(getattr(H, "values", H))):
        return False
    ks = [int(k) for k in ks]
    if any(ks.count(-k) != 1 or ks.count(k) != 1 for k in ks):
        return False
    return int(mode) == int(XMode.convolution) or F.hermitian()


def batch_range(batch: int, rank: int, world: int) -> range:
    a, b = band_ranges(batch, world)[rank]
    return range(a, b)


def gpu_compute(mode, H, T, F, components, inner_dc):
    """Default per-rank compute: the product's sm_100a path, device-resident.
    The signal and the transformation field are uploaded to the rank's current
    CUDA device, xc_run writes the partial sum into a complex64 device tensor
    (XC_DEVICE), and that tensor goes straight into the reduce: no host round
    trip for the partials."""
    import torch
    from . import _native as N
    from .engine import _desc, _param, _signal
    dev = torch.device("cuda", torch.cuda.current_device())
    sig = _signal(H)  # f32 / f64 / c64 / c128 as given (the library converts)
    par = _param(T, sig.shape)  # the steering base keeps the caller's precision
    ds = torch.from_numpy(sig).to(dev)
    dp = torch.from_numpy(par).to(dev)
    out = torch.empty(sig.shape, dtype=torch.complex64, device=dev)
    ctx = N.context(dev.index)
    d = _desc(sig, par, N.XC_C64, T.kind, memory=N.XC_DEVICE)
    comp = np.ascontiguousarray(np.asarray(list(components), np.int32))
    st = N.Stats()
    flags = 0 if inner_dc else N.XC_FLAG_NO_INNER_DC
    torch.cuda.current_stream(dev).synchronize()  # the uploads, before the library's stream
    N.check(N.lib().xc_run(ctx.handle, F.handle(ctx), int(mode), C.byref(d), ds.data_ptr(),
                           dp.data_ptr(),
                           comp.ctypes.data_as(C.POINTER(C.c_int)) if len(comp) else None,
                           len(comp), flags, out.data_ptr(), C.byref(st)), ctx.handle)
    ctx.synchronize()  # the partial is complete before the collective's stream reads it
    return out


def _dist():
    import torch.distributed as dist
    return dist


def _reduce_complex(a, root: int, group=None, device=None):
    """Sum complex partials onto `root` in their own precision.  A CUDA tensor
    (gpu_compute) is reduced where it lies (NCCL over NVLink; gloo, which has
    no CUDA reduce, stages it through host memory); a numpy partial (injected
    CPU compute) is reduced as a CPU tensor, or on `device` if given.  Returns
    the numpy sum on the root, None elsewhere."""
    import torch
    dist = _dist()
    rank = dist.get_rank(group)
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    if not t.is_complex():
        t = t.to(torch.complex128 if t.dtype == torch.float64 else torch.complex64)
    if device is not None:
        t = t.to(device)
    if t.is_cuda and dist.get_backend(group) == "gloo":
        t = t.cpu()
    r = torch.view_as_real(t.contiguous())
    dist.reduce(r, dst=root, op=dist.ReduceOp.SUM, group=group)
    if rank != root:
        return None
    return torch.view_as_complex(r).cpu().numpy()


def _stack(parts):
    import torch
    if all(isinstance(p, torch.Tensor) for p in parts):
        return torch.stack(parts)
    return np.stack([p.cpu().numpy() if isinstance(p, torch.Tensor) else np.asarray(p)
                     for p in parts])


def xfast_band_sharded(mode: XMode, H, T: XformField, F: FreqFilter2,
                       plan: XConvPlan | None = None, compute=gpu_compute, root: int = 0,
                       group=None, device=None) -> Response2 | None:
    """Band-sharded xcorr_fast / xconv_fast; the root returns the Response2."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    plan = plan or XConvPlan()
    ks = list(plan.components) or [int(k) for k in F.ks]
    if world > len(ks):
        raise ValueError("band sharding needs at least one band per rank")
    mine = shard_components(ks, rank, world, shard_in_pairs(mode, H, F, ks))
    inner_dc = rank == root  # add the scale inner-DC term exactly once
    part = compute(int(mode), H, T, F, mine, inner_dc)
    total = _reduce_complex(part, root, group, device)
    if rank != root:
        return None
    out = XConvPlan(mode, T.kind, list(plan.components), plan.periodic)
    return Response2(total, out, len(ks), {})


def _check_integral(F: FreqFilter2) -> None:
    """engine.hpp:388-392: the reconstructed (2R+1)^2 filter must not integrate
    to zero, else the normalization is undefined (same test as xc_smooth)."""
    from .engine import reconstruct
    R = int(np.ceil(F.r_max))
    full = reconstruct(F, 2 * R + 1, 2 * R + 1, float(R), float(R))
    if abs(full.sum()) < 1e-12 * max(1.0, float(np.abs(full).max(initial=0.0))):
        raise ValueError("normalization undefined: filter has zero integral")


def smooth_band_sharded(H, T: XformField, F: FreqFilter2, normalize_signal: bool = True,
                        compute=gpu_compute, root: int = 0, group=None,
                        device=None) -> SmoothResult | None:
    """Band-sharded smooth_adaptive: reduce num and den, divide on the root."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    _check_integral(F)  # engine.hpp:388-392, on every rank before any collective
    # a real image stays real: both scatters then run in conjugate band pairs
    Hs = np.asarray(getattr(H, "values", H))
    Hs = Hs.astype(np.complex128 if np.iscomplexobj(Hs) else np.float64)
    ones = np.ones(Hs.shape, Hs.dtype)
    if normalize_signal and T.kind == XformKind.scale2:  # engine.hpp:396-401
        inv = 1.0 / np.asarray(T.values, np.float64) ** 2
        Hs, ones = Hs * inv, ones * inv
    ks = [int(k) for k in F.ks]
    if world > len(ks):
        raise ValueError("band sharding needs at least one band per rank")
    mine = shard_components(ks, rank, world, shard_in_pairs(XMode.convolution, Hs, F, ks))
    inner_dc = rank == root
    num = compute(int(XMode.convolution), Hs, T, F, mine, inner_dc)
    den = compute(int(XMode.convolution), ones, T, F, mine, inner_dc)
    both = _reduce_complex(_stack([num, den]), root, group, device)
    if rank != root:
        return None
    num, den = both
    floor = 1e-9 * np.max(np.abs(den))  # engine.hpp:408
    bad = np.abs(den) < floor
    out = np.where(bad, 0.0, np.real(num / np.where(bad, 1.0, den)))
    return SmoothResult(out, 2 * len(ks), int(bad.sum()))


# ---------------------------------------------------------------- spatial sharding
# SURVEY 8(e) caveat 3: the angle max is nonlinear across bands, so it shards
# by row strips instead.  G_k(p) = sum_u conj(F_k(u)) H(p + u) only reads rows
# y - R .. y + R (R = ceil(r_max), the render radius, freq_filter.hpp:173-184),
# and the zero padding outside the image is the same for a strip as for the
# whole image, so a strip computed with an R-row halo is the whole-image result
# on its own rows (up to the rounding of a different FFT length).

def strip_rows(h: int, rank: int, world: int, halo: int):
    """(a, b, lo, hi): rank's own rows [a, b) and the halo'd input rows [lo, hi)."""
    a, b = band_ranges(h, world)[rank]
    return a, b, max(0, a - halo), min(h, b + halo)


def gpu_anglemax(H, F, n_angles, components):
    """Default per-rank angle max: the product's sm_100a path."""
    from .engine import anglemax
    return anglemax(H, F, n_angles, components)


def _gather_rows(a: np.ndarray, h: int, root: int, group=None, device=None):
    """Gather every rank's own rows (balanced strips) into the full (h, ...) array
    on the root.  Strips are padded to the largest one so one tensor collective
    (gather; NCCL over NVLink on GPUs) moves them."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    rows = band_ranges(h, world)
    m = max(b - a for a, b in rows)
    buf = np.zeros((m,) + a.shape[1:], a.dtype)
    buf[:a.shape[0]] = a
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    lst = [torch.empty_like(t) for _ in range(world)] if rank == root else None
    dist.gather(t, lst, dst=root, group=group)
    if rank != root:
        return None
    return np.concatenate([lst[r].cpu().numpy()[:b - a] for r, (a, b) in enumerate(rows)])


def _local_peaks(score: np.ndarray, own0: int, own1: int, y0: int, radius: float):
    """Local maxima (vote_filter.hpp:107-134 neighbourhood test, ties broken
    towards the earlier pixel) of the rows [own0, own1) of a strip whose first
    row is image row y0; the strip carries ceil(radius) rows of halo."""
    from .engine import find_peaks
    cand = find_peaks(score, radius, 0.0)  # threshold 0: every local maximum
    return [(p.x, p.y + y0, p.value) for p in cand if own0 <= p.y + y0 < own1]


def anglemax_spatial_sharded(H, F: FreqFilter2, n_angles: int = 360, components=None,
                             compute=gpu_anglemax, root: int = 0, group=None, device=None):
    """Row-strip-sharded angle max; the root returns the full (score, argmax)."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    Hs = np.asarray(H)
    h = Hs.shape[0]
    if world > h:
        raise ValueError("spatial sharding needs at least one row per rank")
    R = int(np.ceil(F.r_max))
    a, b, lo, hi = strip_rows(h, rank, world, R)
    score, arg = compute(np.ascontiguousarray(Hs[lo:hi]), F, n_angles, components)
    score = np.asarray(score)[a - lo:b - lo]
    arg = np.asarray(arg)[a - lo:b - lo]
    s = _gather_rows(np.ascontiguousarray(score), h, root, group, device)
    g = _gather_rows(np.ascontiguousarray(arg), h, root, group, device)
    return None if rank != root else (s, g)


def match_peaks_spatial_sharded(H, F: FreqFilter2, radius: float, threshold_frac: float = 0.5,
                                n_angles: int = 360, components=None, max_peaks: int = 1 << 16,
                                compute=gpu_anglemax, root: int = 0, group=None,
                                device=None):
    """Rotation-invariant matching (angle max + find_peaks, BASELINE config 3)
    on row strips: each rank scores its rows plus a ceil(radius)-row score halo
    (itself computed from an R-row signal halo), keeps the local maxima of its
    own rows, the global max comes from one all-reduce(MAX), and the root merges
    the thresholded candidates with the reference order (value desc, then y,
    then x; vote_filter.hpp:129-132).  The root returns the Peak list."""
    import torch
    from .engine import Peak
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    Hs = np.asarray(H)
    h = Hs.shape[0]
    if world > h:
        raise ValueError("spatial sharding needs at least one row per rank")
    R = int(np.ceil(F.r_max))
    Rn = max(1, int(np.ceil(radius)))
    a, b, slo, shi = strip_rows(h, rank, world, Rn)        # score rows needed
    lo, hi = max(0, slo - R), min(h, shi + R)               # signal rows needed
    score, _ = compute(np.ascontiguousarray(Hs[lo:hi]), F, n_angles, components)
    score = np.ascontiguousarray(np.asarray(score)[slo - lo:shi - lo])
    own = score[a - slo:b - slo]
    mx = torch.tensor([float(own.max()) if own.size else -np.inf], dtype=torch.float64)
    if device is not None:
        mx = mx.to(device)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    thresh = threshold_frac * float(mx.item())
    mine = [c for c in _local_peaks(score, a, b, slo, radius) if not c[2] < thresh]
    allc = [None] * world
    dist.all_gather_object(allc, mine, group=group)
    if rank != root:
        return None
    peaks = sorted((c for part in allc for c in part), key=lambda c: (-c[2], c[1], c[0]))
    return [Peak(int(x), int(y), float(v)) for x, y, v in peaks[:max_peaks]]
