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

import numpy as np

from .engine import (FreqFilter2, Response2, SmoothResult, XConvPlan, XformField, XformKind,
                     XMode, _fast)


def band_ranges(n: int, world: int):
    """Contiguous ranges balanced to +-1 (65 bands over 8 ranks: 9,8,...,8)."""
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


def shard_components(ks, rank: int, world: int) -> list:
    ks = [int(k) for k in ks]
    a, b = band_ranges(len(ks), world)[rank]
    return ks[a:b]


def batch_range(batch: int, rank: int, world: int) -> range:
    a, b = band_ranges(batch, world)[rank]
    return range(a, b)


def gpu_compute(mode, H, T, F, components, inner_dc):
    """Default per-rank compute: the product's sm_100a path."""
    return _fast(XMode(mode), H, T, F, XConvPlan(components=list(components)),
                 inner_dc=inner_dc).output


def _dist():
    import torch.distributed as dist
    return dist


def _reduce_complex(a: np.ndarray, root: int, group=None, device=None) -> np.ndarray:
    import torch
    dist = _dist()
    t = torch.from_numpy(np.ascontiguousarray(a.astype(np.complex128)))
    t = torch.view_as_real(t).contiguous()
    if device is not None:
        t = t.to(device)
    dist.reduce(t, dst=root, op=dist.ReduceOp.SUM, group=group)
    return torch.view_as_complex(t.cpu().contiguous()).numpy()


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
    mine = shard_components(ks, rank, world)
    inner_dc = rank == root  # add the scale inner-DC term exactly once
    part = compute(int(mode), H, T, F, mine, inner_dc)
    total = _reduce_complex(np.asarray(part), root, group, device)
    if rank != root:
        return None
    out = XConvPlan(mode, T.kind, list(plan.components), plan.periodic)
    return Response2(total, out, len(ks), {})


def smooth_band_sharded(H, T: XformField, F: FreqFilter2, normalize_signal: bool = True,
                        compute=gpu_compute, root: int = 0, group=None,
                        device=None) -> SmoothResult | None:
    """Band-sharded smooth_adaptive: reduce num and den, divide on the root."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    Hs = np.asarray(H, np.complex128)
    ones = np.ones(Hs.shape, np.complex128)
    if normalize_signal and T.kind == XformKind.scale2:  # engine.hpp:396-401
        inv = 1.0 / np.asarray(T.values, np.float64) ** 2
        Hs, ones = Hs * inv, ones * inv
    ks = [int(k) for k in F.ks]
    if world > len(ks):
        raise ValueError("band sharding needs at least one band per rank")
    mine = shard_components(ks, rank, world)
    inner_dc = rank == root
    num = np.asarray(compute(int(XMode.convolution), Hs, T, F, mine, inner_dc))
    den = np.asarray(compute(int(XMode.convolution), ones, T, F, mine, inner_dc))
    both = _reduce_complex(np.stack([num, den]), root, group, device)
    if rank != root:
        return None
    num, den = both
    floor = 1e-9 * np.max(np.abs(den))  # engine.hpp:408
    bad = np.abs(den) < floor
    out = np.where(bad, 0.0, np.real(num / np.where(bad, 1.0, den)))
    return SmoothResult(out, 2 * len(ks), int(bad.sum()))
