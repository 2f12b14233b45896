#!/usr/bin/env python
"""Benchmark of the B200 extended-correlation hot path (BASELINE.json metric).

Workload (default): BASELINE config 5 -- a batch of 16 images of 4096 x 4096
fp32, 63 x 63 filter with |m| <= 32 (65 rotation bands), per-pixel angle
theta ~ U[0, 2 pi), extended correlation (gather).  One step = xcorr_fast over
the whole batch.  Metric: Mpixel.bands/s = H*W*standard_ops*images / time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

--config 1..5 selects another BASELINE config (2: scatter, 3: 360-angle max,
4: smoothing); each prints the same line with the roofline of its dominant
kernel.  Multi-GPU: the 16 images are sharded across ranks (no data-path
collective); --shard bands instead uses a rank context of the C ABI
(xc_context_create_rank): every rank computes its band range and the library
sums the partial outputs with an NCCL reduce that overlaps the next step
(XC_FLAG_ASYNC).  `value` is device-timed with inputs resident in HBM; `e2e`
times the public API with pinned host buffers (H2D + D2H inside the region).
`--impl reference` times the reference itself (oracle/_ref: its headers
compiled unchanged against an Eigen-subset shim) on all host cores.
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


def peaks_all() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


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

    def sample_now(self):
        """One synchronous sample (a timed region shorter than the 100 ms
        sampling period leaves none)."""
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=30).stdout
            for line in out.splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 6:
                    self.rows.append(parts)
                    self.after_region = True
        except (OSError, subprocess.SubprocessError):
            pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
               "samples": len(self.rows)}
        if getattr(self, "after_region", False):
            out["note"] = "timed region shorter than the sampling period: sampled right after it"
        return out


def stage_bytes(stage: str, B: int, H: int, W: int, Ph: int, Pw: int, ni: int = 1,
                spectra: int | None = None, t2_planes: int = 1) -> float:
    """Algorithmic bytes of one launch of each pipeline stage covering `ni`
    images: the compulsory reads + writes of its inputs/outputs (complex fp32 =
    8 B; B = bands the stage transforms).  I1 reads each filter spectrum once
    per launch (shared by its images).  The scatter's conjugate band pairs
    (xc_stats.band_mode 2) transform B = the bands k >= 0 but S2 still reads
    `spectra` = every band's spectrum and writes t2_planes = 2 sums."""
    N, P = H * W, Ph * Pw
    H2, Hx2 = H + (H & 1), H + (H & 1)
    S = B if spectra is None else spectra
    if stage == "I1_cols_inv_corr":
        return ni * (8 * P + B * 8 * H2 * Pw) + B * 8 * P
    return ni * {
        "prep": 4 * N + 8 * N,
        "F1_rows_fwd": 4 * N + 8 * Hx2 * Pw,
        "F2_cols_fwd": 8 * Hx2 * Pw + 8 * P,
        "I2_rows_inv_steer": B * 8 * H2 * Pw + 8 * N + 8 * N,
        "I2_rows_inv_planes": B * 8 * H2 * Pw + B * 8 * N,
        "anglemax": B * 8 * N + 4 * N + 4 * N,
        "S1_rows_fwd_premul": 4 * N + 8 * N + B * 8 * Hx2 * Pw,
        "S2_cols_fwd_mac_inv": B * 8 * Hx2 * Pw + S * 8 * P + t2_planes * 8 * H2 * Pw,
        "S4_rows_inv_out": t2_planes * 8 * H2 * Pw + 8 * N,
        "smooth_finish": 8 * N + 8 * N + 4 * N,
        "absmax": 4 * N,
    }.get(stage, float("nan"))


def model_bytes(mode: str, B: int, N: int, P: int) -> float:
    """SURVEY 8(d) per-image algorithmic-bytes model of the whole pipeline."""
    if mode == "xcorr":
        return 16 * N + 8 * P + B * (16 * P + 16 * N)
    if mode == "anglemax":
        return 12 * N + 8 * P + B * (16 * P + 16 * N)
    scatter = 16 * N + 16 * P + 24 * B * P
    return 2 * scatter + 20 * N if mode == "smooth" else scatter


MODES = {1: "xcorr", 2: "xconv", 3: "anglemax", 4: "smooth", 5: "xcorr"}


def host_info() -> str:
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in out.splitlines()
                      if ln.startswith("Model name")), "")
    except OSError:
        pass
    return f"nproc {os.cpu_count()}, {model or 'unknown CPU'}"


def ref_backend():
    """The reference itself (oracle/_ref, kind 'reference') when built, else the
    oracle restatement (kind 'port')."""
    from oracle import refimpl
    if refimpl.available():
        return refimpl, "reference"
    from oracle import oracle as orc
    return orc, "port"


def cpu_sample(w, nthreads: int, nbands: int):
    """One bounded CPU sample of the workload's per-band loop (engine.hpp:300
    / 345): the reference (or the port) on image 0 with `nbands` bands split
    across `nthreads` threads.  Returns (seconds, pixel.bands, kind)."""
    mod, kind = ref_backend()
    F = w.filt if getattr(w.filt, "__module__", "").startswith("oracle") else None
    if F is None:  # a product filter: rebuild it with the backend's own decomposition
        group, args = w.decomp
        F = (mod.decompose_rotation2 if group == "rotation2" else mod.decompose_scale2)(
            w.filter_image, *args)
    H = w.signal[0].astype(np.float64)
    if w.param is None:  # angle max: the per-band correlations G_k (unsteered)
        T, xk, mode = np.zeros_like(H), 0, 0
    else:
        T, xk, mode = w.param[0].astype(np.float64), int(w.kind), (0 if w.mode == "xcorr" else 1)
    ks = [int(k) for k in F.ks[:nbands]]
    t0 = time.perf_counter()
    if kind == "reference":
        _, ops = mod.xfast(mode, H, xk, T, F, components=ks, nthreads=nthreads)
    else:
        fn = mod.xcorr_fast if mode == 0 else mod.xconv_fast
        ops = fn(H, xk, T, F, components=ks, nthreads=nthreads)[1]
    dt = time.perf_counter() - t0
    return dt, H.size * ops, kind


def make_workload(cfg: int, small: bool, backend=None):
    from paper_2006_13188_b200 import workloads as WL
    if cfg == 5:
        return WL.config5(n=512 if small else 4096, batch=16, backend=backend)
    kw = {"n": 256} if small else {}
    return WL.CONFIGS[cfg](backend=backend, **kw)


def run_reference(args):
    """The reference's own CPU implementation of the path (oracle/_ref: its
    headers compiled unchanged) on all host threads, on this arm's config: each
    step is a bounded sample -- image 0 with one band per thread, the bands
    split across threads (the reference's band loop is independent per band,
    engine.hpp:300) -- and the value is its pixel.band throughput, which the
    per-band, per-image loop makes exact to extrapolate to the whole job."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    mod, kind = ref_backend()
    w = make_workload(args.config, args.small, backend=mod)  # no product library loaded
    nthreads = max(1, min(os.cpu_count() or 1, 64))
    nb = min(nthreads, w.bands)
    for _ in range(args.warmup):
        cpu_sample(w, nthreads, nb)
    ts = []
    units = 0
    for _ in range(args.steps):
        dt, units, kind = cpu_sample(w, nthreads, nb)
        ts.append(dt)
    t = sum(ts) / len(ts)
    value = units / t / 1e6
    B, H, W = w.signal.shape
    what = {"xcorr": "xcorr_fast", "xconv": "xconv_fast (smooth_adaptive runs two of these)",
            "smooth": "xconv_fast (smooth_adaptive runs two of these)",
            "anglemax": "single-band xcorr_fast (the G_k of the angle max)"}[w.mode]
    sample = (f"{'the reference (oracle/_ref, its own headers compiled unchanged)' if kind == 'reference' else 'the oracle port'}"
              f" {what} on image 0 of {w.name} ({H}x{W}), {nb} of {w.bands} bands per step "
              f"on {nthreads} threads, double precision; extrapolated per pixel.band to the "
              f"{B}-image job (the band loop engine.hpp:300 is per band and per image); "
              f"{host_info()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config)",
        "config": {"workload": w.name, "images": int(B), "height": int(H), "width": int(W),
                   "bands": w.bands},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def hermitian(F) -> bool:
    """HostFilter::hermitian(): F_{-k} = conj(F_k) within 1e-12 of the largest
    coefficient (the library's half-band test)."""
    ks = list(np.asarray(F.ks))
    c = np.asarray(F.comps)
    tol = 1e-12 * max(np.abs(c).max(initial=0.0), 1e-300)
    for i, k in enumerate(ks):
        if -k not in ks or np.abs(c[:, ks.index(-k)] - np.conj(c[:, i])).max() > tol:
            return False
    return True


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
    mode = MODES[args.config]
    Btot, H, W = w.signal.shape
    F = w.filt
    nb = F.n_components()
    ops_per_image = nb * (2 if mode == "smooth" else 1)
    shard = args.shard
    if world > 1 and shard == "batch" and Btot < world:
        shard = "replicas"  # SURVEY 8(e) caveat 5: fewer images than ranks
    if shard == "bands" and mode == "anglemax":
        raise SystemExit("the angle max is nonlinear across bands: use --shard batch "
                         "(spatial sharding lives in paper_2006_13188_b200.distributed)")
    if shard == "bands" and world > nb:
        raise SystemExit(f"band sharding needs at least one band per rank ({nb} bands, "
                         f"{world} ranks)")
    if world > 1 and shard == "batch":
        imgs = list(range(rank * Btot // world, (rank + 1) * Btot // world))
    else:
        imgs = list(range(Btot))
    Bl = len(imgs)
    band_mode = shard == "bands" and use_dist
    if band_mode:
        # the library shards the bands and reduces with NCCL (xc_context_create_rank)
        ids = [N.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        ctx = N.Context.rank(local, ids[0], rank, world)
    else:
        ctx = N.context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    fh = F.handle()
    # inputs resident in HBM (the workload's own seeded arrays, uploaded once)
    sig = torch.from_numpy(w.signal[imgs[0]:imgs[-1] + 1]).to(dev)
    par = torch.from_numpy(w.param[imgs[0]:imgs[-1] + 1]).to(dev) if w.param is not None else None
    if mode in ("xcorr", "xconv"):
        out_dt, odt = N.XC_C64, torch.complex64
    else:
        out_dt, odt = N.XC_F32, torch.float32
    outs = [torch.empty((Bl, H, W), dtype=odt, device=dev) for _ in range(2 if band_mode else 1)]
    arg = torch.empty((Bl, H, W), dtype=torch.int32, device=dev) if mode == "anglemax" else None
    flags = N.XC_FLAG_ASYNC if band_mode else 0
    kind = int(F.group)
    st = N.Stats()

    def call(desc, s_ptr, p_ptr, o_ptr, fl):
        if mode in ("xcorr", "xconv"):
            rc = N.lib().xc_run(ctx.handle, fh, 0 if mode == "xcorr" else 1, C.byref(desc),
                                C.c_void_p(s_ptr), C.c_void_p(p_ptr), None, 0, fl,
                                C.c_void_p(o_ptr), C.byref(st))
        elif mode == "smooth":
            rc = N.lib().xc_smooth(ctx.handle, fh, C.byref(desc), C.c_void_p(s_ptr),
                                   C.c_void_p(p_ptr), 1, C.c_void_p(o_ptr), C.byref(st))
        else:
            rc = N.lib().xc_anglemax(ctx.handle, fh, C.byref(desc), C.c_void_p(s_ptr), None, 0,
                                     360, C.c_void_p(o_ptr),
                                     C.cast(C.c_void_p(a_ptr[0]), C.POINTER(C.c_int)),
                                     C.byref(st))
        N.check(rc, ctx.handle)
        return st.gpu_launches

    a_ptr = [arg.data_ptr() if arg is not None else 0]
    dd = N.ImageDesc(H, W, Bl, N.XC_F32, N.XC_F32, out_dt, N.XC_ROW_MAJOR, N.XC_DEVICE, 1, kind)
    step_no = [0]

    def step_device():
        o = outs[step_no[0] % len(outs)]
        step_no[0] += 1
        return call(dd, sig.data_ptr(), par.data_ptr() if par is not None else 0, o.data_ptr(),
                    flags)

    def drain():
        if band_mode:
            ctx.synchronize()  # the queued band reduces

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step_device()
    drain()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step_device()
    drain()
    e1.record(stream)
    barrier()
    # stage events inside the timed region when a step is long enough not to
    # be perturbed by them; short (launch-bound) steps get a separate profiled
    # pass of the same steps for the per-kernel roofline
    in_region = e0.elapsed_time(e1) > 2.0
    # short (launch-bound) rotation steps replay a CUDA graph of the call:
    # XC_FLAG_ASYNC with device memory leaves the kernels queued on the
    # context's stream, so the whole launch sequence is captured once
    graphed = not in_region and not band_mode and mode in ("xcorr", "xconv") and kind == 0
    if graphed:
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            ctx.set_stream(cap.cuda_stream)
            graph_launches = call(dd, sig.data_ptr(), par.data_ptr(), outs[0].data_ptr(),
                                  N.XC_FLAG_ASYNC)
        ctx.set_stream(stream.cuda_stream)
        plain_step = step_device

        def step_device():
            graph.replay()
            return graph_launches

        for _ in range(args.warmup):
            step_device()
        barrier()
    if in_region:
        ctx.profile(enable=True, reset=True)
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            launches += step_device()
        drain()
        e1.record(stream)
        barrier()
    if not clk.rows:
        clk.sample_now()
    if not in_region:
        ctx.profile(enable=True, reset=True)
        for _ in range(args.steps):
            (plain_step if graphed else step_device)()
        drain()
        barrier()
    prof = ctx.profile(enable=False, reset=True)
    nb_run = st.bands_run or nb
    cpair = st.band_mode == 2  # scatter of a real signal: conjugate band pairs
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    job_images = Btot * (world if shard == "replicas" else 1)
    units_step = job_images * H * W * ops_per_image
    value = units_step / (ms_step * 1e-3) / 1e6

    # ---- e2e: public API with pinned host buffers (H2D + D2H in the region)
    e2e = None
    if not args.no_e2e:
        hsig = torch.from_numpy(w.signal[imgs[0]:imgs[-1] + 1]).pin_memory()
        hpar = (torch.from_numpy(w.param[imgs[0]:imgs[-1] + 1]).pin_memory()
                if w.param is not None else None)
        hout = torch.empty((Bl, H, W), dtype=odt).pin_memory()
        if arg is not None:
            harg = torch.empty((Bl, H, W), dtype=torch.int32).pin_memory()
            a_ptr[0] = harg.data_ptr()
        dh = N.ImageDesc(H, W, Bl, N.XC_F32, N.XC_F32, out_dt, N.XC_ROW_MAJOR, N.XC_HOST, 1, kind)

        def step_host():
            call(dh, hsig.data_ptr(), hpar.data_ptr() if hpar is not None else 0,
                 hout.data_ptr(), 0)

        step_host()
        barrier()
        # wall-clock region: short steps (< 5 ms) run every step, long ones up to 3
        n_e2e = max(1, args.steps if ms_step < 5.0 else min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            step_host()
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / n_e2e], device=dev, dtype=torch.float64)
        if use_dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        in_bytes = Bl * H * W * (4 + (4 if w.param is not None else 0))
        out_bytes = Bl * H * W * (odt.itemsize + (4 if arg is not None else 0))
        ranks_in = world if use_dist else 1  # every rank uploads its own inputs
        ranks_out = 1 if band_mode else ranks_in  # band mode: rank 0 receives the sum
        e2e = {"value": units_step / float(te.item()) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(in_bytes * ranks_in),
               "d2h_bytes_per_step": int(out_bytes * ranks_out), "steps": n_e2e}

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (CUDA events around each stage)
    hbm, peak_kind = peaks()
    Ph, Pw = st.pad_h, st.pad_w
    dom = max(prof, key=lambda k: prof[k][0]) if prof else None
    roof = None

    def kernel_roof(name):
        tot_ms, nl = prof[name]
        per_launch_s = tot_ms * 1e-3 / nl
        ni = max(1, round(Bl * args.steps / nl))  # images per launch
        alg = stage_bytes(name, nb_run, H, W, Ph, Pw, ni, nb if cpair else None,
                          2 if cpair else 1)
        return alg, per_launch_s, ni, alg / per_launch_s / 1e9

    # committed ncu --set full per-launch statistics (tools/ncu_stats.py)
    kstats = {}
    sf = os.path.join(ROOT, "profiles", "ncu_kernel_stats.json")
    if os.path.exists(sf):
        with open(sf) as f:
            kstats = json.load(f)
    clk_now = clk.summary()
    sm_mhz = clk_now.get("sm_mhz") or clk_now.get("sm_max_mhz") or 1965.0
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count

    def issue_roof(name, per_launch_s):
        """The instruction-issue roofline: ncu's warp instructions per launch of
        this kernel (same code, same config) over the live launch time at the
        sampled SM clock, against one warp instruction per cycle per SMSP."""
        ks = kstats.get(f"cfg{args.config}:{name}")
        if not ks or not ks.get("warp_instructions"):
            return None
        peak = 4 * n_sm * sm_mhz * 1e6  # warp instructions / s
        ach = ks["warp_instructions"] / per_launch_s
        return {"warp_instructions_per_launch": ks["warp_instructions"], "achieved": ach,
                "peak": peak, "unit": "warp inst/s", "frac": ach / peak,
                "sm_mhz": sm_mhz, "source": ks.get("source")}

    def tensor_roof(name, per_launch_s):
        """The angle max runs on the tensor cores (k_anglemax_tc.cu, config 3):
        12 tf32 MMAs of 128 x 192 x 8 per 128-pixel tile (3xTF32 split), against
        the dense tf32 peak = half the measured bf16 peak."""
        if name != "anglemax" or os.environ.get("XCB_ANGLE_TC") == "0":
            return None
        ntiles = -(-H * W // 128) * max(1, round(Bl * args.steps / prof[name][1]))
        flops = ntiles * 12 * 2 * 128 * 192 * 8
        pk = peaks_all().get("bf16_tflops")
        if not pk:
            return None
        ach = flops / per_launch_s / 1e12
        return {"kernel": "k_anglemax_tc", "executed_tflop_per_launch": flops / 1e12,
                "achieved": ach, "peak": pk / 2, "unit": "TFLOP/s (tf32)", "frac": ach / (pk / 2),
                "note": "3xTF32: a third of the executed flops are the fp32-equivalent sums"}

    if dom:
        alg, per_launch_s, ni, achieved = kernel_roof(dom)
        ks = kstats.get(f"cfg{args.config}:{dom}")
        traffic = ks["dram_bytes"] * ni if ks and ks.get("dram_bytes") else None
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_kind,
                "alg_bytes_per_launch": alg, "ms_per_launch": per_launch_s * 1e3,
                "images_per_launch": ni, "bands_transformed": nb_run,
                "band_mode": {0: "all bands", 1: "hermitian half-band",
                              2: "conjugate band pairs"}.get(st.band_mode),
                "stage_events": "in the timed region" if in_region else
                                "separate profiled pass of the same steps (short steps)",
                "cuda_graph": graphed,
                "issue": issue_roof(dom, per_launch_s),
                "tensor": tensor_roof(dom, per_launch_s),
                "kernels": {k: {"ms_per_launch": kernel_roof(k)[1] * 1e3,
                                "images_per_launch": kernel_roof(k)[2],
                                "achieved_gbs": kernel_roof(k)[3],
                                "frac": kernel_roof(k)[3] / hbm,
                                "issue_frac": (issue_roof(k, kernel_roof(k)[1]) or {}).get("frac")}
                            for k in prof if k != "prep"},
                "stages_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
                "pipeline_model_frac": model_bytes(mode, nb, H * W, Ph * Pw) * Bl /
                (ms_step * 1e-3) / 1e9 / hbm}
        if roof["tensor"]:  # the dominant kernel is the tensor-core angle max
            tr = roof["tensor"]
            roof["hbm_view"] = {k: roof[k] for k in ("achieved", "peak", "unit", "frac")}
            roof.update({"bound": "tensor", "achieved": tr["achieved"], "peak": tr["peak"],
                         "unit": "TFLOP/s", "frac": tr["frac"]})

    cpu = None
    if world == 1 and not args.no_cpu:
        dt, u, ck = cpu_sample(w, 1, 2)
        cpu = {"value": u / dt / 1e6, "unit": UNIT, "cores": 1, "kind": ck,
               "sample": f"{'the reference (oracle/_ref)' if ck == 'reference' else 'the oracle port'}"
                         f" on image 0 of {w.name}, 2 of {nb} bands, 1 thread, double "
                         f"precision, {dt:.1f} s; {host_info()}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if shard in ("batch", "bands") else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy, BASELINE config; uploaded to HBM before timing)",
        "config": {"workload": w.name, "mode": mode, "images": Btot, "height": H, "width": W,
                   "bands": nb, "pad": [Ph, Pw],
                   "shard": shard if use_dist else "none",
                   "l2": "inputs larger than L2 (%.2f GB read per step)"
                         % (Bl * H * W * 8 / 1e9) if Bl * H * W * 8 > 126e6 else
                         "inputs L2-resident (launch-bound config)"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "cuda_graph": graphed,
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
