#!/usr/bin/env python
"""Benchmark of the B200 extended-correlation hot path (BASELINE.json metric).

Workload (default): BASELINE config 5 -- a batch of 16 images of 4096 x 4096
fp32, 63 x 63 filter with |m| <= 32 (65 rotation bands), per-pixel angle
theta ~ U[0, 2 pi), extended correlation (gather).  One step = xcorr_fast over
the whole batch.  Metric: Mpixel.bands/s = H*W*standard_ops*images / time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Multi-GPU: the 16 images are sharded across ranks (no data-path collective;
--shard bands instead splits the 65 bands and sums the partial outputs with an
NCCL reduce).  `value` is device-timed with inputs resident in HBM; `e2e`
times the public API with pinned host buffers (H2D + D2H inside the region).
`--impl reference` times the CPU oracle (the reference restated; the
reference itself cannot be built here) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "extended correlation Mpixel·bands/s at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Mpixel·bands/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def stage_bytes(stage: str, B: int, H: int, W: int, Ph: int, Pw: int, ni: int = 1) -> float:
    """Algorithmic bytes of one launch of each pipeline stage covering `ni`
    images: the compulsory reads + writes of its inputs/outputs (complex fp32 =
    8 B).  I1 reads each filter spectrum once per launch (shared by its images)."""
    N, P = H * W, Ph * Pw
    H2, Hx2 = H + (H & 1), H + (H & 1)
    if stage == "I1_cols_inv_corr":
        return ni * (8 * P + B * 8 * H2 * Pw) + B * 8 * P
    return ni * {
        "prep": 4 * N + 8 * N,
        "F1_rows_fwd": 4 * N + 8 * Hx2 * Pw,
        "F2_cols_fwd": 8 * Hx2 * Pw + 8 * P,
        "I2_rows_inv_steer": B * 8 * H2 * Pw + 8 * N + 8 * N,
        "S1_rows_fwd_premul": 4 * N + 8 * N + B * 8 * Hx2 * Pw,
        "S2_cols_fwd_mac_inv": B * 8 * Hx2 * Pw + B * 8 * P + 8 * H2 * Pw,
        "S4_rows_inv_out": 8 * H2 * Pw + 8 * N,
    }.get(stage, float("nan"))


def model_bytes(mode: str, B: int, N: int, P: int) -> float:
    """SURVEY 8(d) per-image algorithmic-bytes model of the whole pipeline."""
    if mode == "xcorr":
        return 16 * N + 8 * P + B * (16 * P + 16 * N)
    return 16 * N + 16 * P + 24 * B * P


def cpu_sample(w, nthreads: int, nbands: int):
    """Time the CPU oracle on image 0 with `nbands` bands; returns (s, units)."""
    from oracle import oracle as orc
    F = orc.Filter(int(w.filt.group), w.filt.K, w.filt.ks, w.filt.comps, w.filt.n_radii,
                   w.filt.n_angles, w.filt.r_max, w.filt.r_min, w.filt.r_domain)
    H = w.signal[0].astype(np.float64)
    T = w.param[0].astype(np.float64)
    ks = [int(k) for k in w.filt.ks[:nbands]]
    t0 = time.perf_counter()
    _, ops, _ = orc.xcorr_fast(H, 0, T, F, components=ks, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return dt, H.size * ops


def make_workload(cfg: int, small: bool):
    from paper_2006_13188_b200 import workloads as WL
    if cfg == 5:
        return WL.config5(n=512 if small else 4096, batch=16)
    return WL.CONFIGS[cfg](**({"n": 256} if small else {}))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = make_workload(args.config, args.small)
    nthreads = max(1, min(os.cpu_count() or 1, 32))
    nb = min(nthreads, w.bands)
    for _ in range(args.warmup):
        cpu_sample(w, nthreads, nb)
    ts = []
    units = 0
    for _ in range(args.steps):
        dt, units = cpu_sample(w, nthreads, nb)
        ts.append(dt)
    t = sum(ts) / len(ts)
    value = units / t / 1e6
    sample = (f"image 0 of {w.name} ({w.signal.shape[1]}x{w.signal.shape[2]}), {nb} of "
              f"{w.bands} bands per step, double precision, reference structure (3 FFTs per band)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config)",
        "config": {"workload": w.name, "images": int(w.signal.shape[0]),
                   "height": int(w.signal.shape[1]), "width": int(w.signal.shape[2]),
                   "bands": w.bands},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # under torchrun (even with one rank) the NCCL plumbing runs: process
    # group, barriers, the band reduce and the max-over-ranks timing
    use_dist = world > 1 or "LOCAL_WORLD_SIZE" in os.environ or "TORCHELASTIC_RUN_ID" in os.environ
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2006_13188_b200 import _native as N
    import ctypes as C
    w = make_workload(args.config, args.small)
    if w.mode != "xcorr":
        raise SystemExit("bench.py measures the extended-correlation configs (1, 5)")
    Btot, H, W = w.signal.shape
    F = w.filt
    nb = F.n_components()
    ks = np.asarray(F.ks, np.int32)
    # fewer images than ranks (config 1): every rank runs a replica of the
    # whole batch ("replicas only"), and the job's units scale
    replicas = args.shard == "batch" and world > 1 and Btot < world
    if args.shard == "batch" and world > 1 and not replicas:
        imgs = list(range(rank * Btot // world, (rank + 1) * Btot // world))
        comps = ks
    elif replicas:
        imgs = list(range(Btot))
        comps = ks
    else:
        imgs = list(range(Btot))
        comps = ks[rank * nb // world:(rank + 1) * nb // world] if world > 1 else ks
    Bl = len(imgs)
    # inputs resident in HBM (the workload's own seeded arrays, uploaded once)
    sig = torch.from_numpy(w.signal[imgs[0]:imgs[-1] + 1]).to(dev)
    th = torch.from_numpy(w.param[imgs[0]:imgs[-1] + 1]).to(dev)
    out = torch.empty((Bl, H, W), dtype=torch.complex64, device=dev)
    ctx = N.context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    fh = F.handle()
    cptr = np.ascontiguousarray(comps)
    flags = 0
    if args.shard == "bands" and world > 1 and rank != 0 and F.group == 1:
        flags |= N.XC_FLAG_NO_INNER_DC
    dd = N.ImageDesc(H, W, Bl, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_DEVICE, 1,
                     int(F.group))
    st = N.Stats()

    # band sharding: the reduce of step i runs on NCCL's stream while step
    # i + 1 computes into the other output buffer (overlap each
    # reduce with the next compute); drain() joins the outstanding reduces
    band_reduce = args.shard == "bands" and use_dist
    outs = [out, torch.empty_like(out)] if band_reduce else [out]
    pending = [None] * len(outs)
    step_no = [0]

    def step_device():
        i = step_no[0] % len(outs)
        step_no[0] += 1
        if pending[i] is not None:
            pending[i].wait()
            pending[i] = None
        N.check(N.lib().xc_run(ctx.handle, fh, 0, C.byref(dd), C.c_void_p(sig.data_ptr()),
                               C.c_void_p(th.data_ptr()), cptr.ctypes.data_as(C.POINTER(C.c_int)),
                               len(cptr), flags, C.c_void_p(outs[i].data_ptr()), C.byref(st)),
                ctx.handle)
        if band_reduce:
            pending[i] = dist.reduce(outs[i], dst=0, op=dist.ReduceOp.SUM, async_op=True)
        return st.gpu_launches

    def drain():
        for i, p in enumerate(pending):
            if p is not None:
                p.wait()
                pending[i] = None

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step_device()
    drain()
    barrier()
    ctx.profile(enable=True, reset=True)
    launches = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            launches += step_device()
        drain()
        e1.record(stream)
        barrier()
    prof = ctx.profile(enable=False, reset=True)
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    units_step = Btot * H * W * nb * (world if replicas else 1)
    value = units_step / (ms_step * 1e-3) / 1e6

    # ---- e2e: public API with pinned host buffers (H2D + D2H in the region)
    e2e = None
    if not args.no_e2e:
        hsig = torch.from_numpy(w.signal[imgs[0]:imgs[-1] + 1]).pin_memory()
        hth = torch.from_numpy(w.param[imgs[0]:imgs[-1] + 1]).pin_memory()
        hout = torch.empty((Bl, H, W), dtype=torch.complex64).pin_memory()
        dh = N.ImageDesc(H, W, Bl, N.XC_F32, N.XC_F32, N.XC_C64, N.XC_ROW_MAJOR, N.XC_HOST, 1,
                         int(F.group))

        def step_host():
            N.check(N.lib().xc_run(ctx.handle, fh, 0, C.byref(dh), C.c_void_p(hsig.data_ptr()),
                                   C.c_void_p(hth.data_ptr()),
                                   cptr.ctypes.data_as(C.POINTER(C.c_int)), len(cptr), flags,
                                   C.c_void_p(hout.data_ptr()), C.byref(st)), ctx.handle)

        step_host()
        barrier()
        n_e2e = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            step_host()
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / n_e2e], device=dev, dtype=torch.float64)
        if use_dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": units_step / float(te.item()) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(Btot * H * W * 8 * (world if replicas else 1)),
               "d2h_bytes_per_step": int(Btot * H * W * 8 * (world if replicas else 1)),
               "steps": n_e2e}

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (CUDA events around each stage)
    hbm, peak_kind = peaks()
    Ph, Pw = st.pad_h, st.pad_w
    dom = max(prof, key=lambda k: prof[k][0]) if prof else None
    roof = None
    nbl = len(comps)

    def kernel_roof(name):
        tot_ms, nl = prof[name]
        per_launch_s = tot_ms * 1e-3 / nl
        ni = max(1, round(Bl * args.steps / nl))  # images per launch
        alg = stage_bytes(name, nbl, H, W, Ph, Pw, ni)
        return alg, per_launch_s, ni, alg / per_launch_s / 1e9

    if dom:
        alg, per_launch_s, ni, achieved = kernel_roof(dom)
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):
            with open(tf) as f:
                traffic = json.load(f).get(f"cfg{args.config}:{dom}")
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_kind,
                "alg_bytes_per_launch": alg, "ms_per_launch": per_launch_s * 1e3,
                "images_per_launch": ni,
                "kernels": {k: {"ms_per_launch": kernel_roof(k)[1] * 1e3,
                                "images_per_launch": kernel_roof(k)[2],
                                "achieved_gbs": kernel_roof(k)[3],
                                "frac": kernel_roof(k)[3] / hbm}
                            for k in prof if k.startswith("I")},
                "stages_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
                "pipeline_model_frac": model_bytes("xcorr", nb, H * W, Ph * Pw) * Btot *
                (world if replicas else 1) /
                (ms_step * 1e-3) / 1e9 / hbm / max(world, 1)}

    cpu = None
    if world == 1 and not args.no_cpu:
        dt, u = cpu_sample(w, 1, 2)
        cpu = {"value": u / dt / 1e6, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"image 0 of {w.name}, 2 of {nb} bands, 1 thread, double precision, "
                         f"reference structure (3 FFTs per band), {dt:.1f} s"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy, BASELINE config; uploaded to HBM before timing)",
        "config": {"workload": w.name, "images": Btot, "height": H, "width": W, "bands": nb,
                   "pad": [Ph, Pw],
                   "shard": ("replicas" if replicas else args.shard) if use_dist else "none",
                   "l2": "inputs larger than L2 (signal + theta %.1f GB per step)"
                         % (Btot * H * W * 8 / 1e9)},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--shard", default="batch", choices=["batch", "bands"])
    ap.add_argument("--small", action="store_true", help="reduced sizes (smoke)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
