"""Spatially sharded matching on the GPU path (SURVEY 8(e) caveat 3): two gloo
ranks, each running its row strip (with halos) through the sm_100a angle max on
cuda:0, merge peaks equal to the single-process peaks.  The ranks' kernels are
independent (the exchange is gloo on host tensors), so sharing one GPU does not
make them wait on each other."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_13188_b200 import distributed as D
    from paper_2006_13188_b200 import workloads as WL
    w = WL.config3(n=640, n_templates=3)
    pk = D.match_peaks_spatial_sharded(w.signal[0], w.filt, 32.0, 0.5, 360)
    sc = D.anglemax_spatial_sharded(w.signal[0], w.filt, 360)
    if rank == 0:
        q.put({"peaks": [(p.x, p.y, p.value) for p in pk], "score": sc[0]})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_spatial_sharded_matching_gpu_world2():
    import paper_2006_13188_b200 as X
    from paper_2006_13188_b200 import workloads as WL
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = WL.config3(n=640, n_templates=3)
    score, _ = X.anglemax(w.signal[0], w.filt, 360)
    rel = np.linalg.norm(res["score"] - score) / np.linalg.norm(score)
    assert rel < 1e-5
    ref = X.find_peaks(score.astype(np.float64), 32.0, 0.5)
    got = res["peaks"]
    assert len(got) >= 3
    assert [(x, y) for x, y, _ in got[:3]] == [(p.x, p.y) for p in ref[:3]]
    for (cx, cy, _), (x, y, _) in zip(sorted(w.meta["truth"]), sorted(got[:3])):
        assert abs(x - cx) <= 2 and abs(y - cy) <= 2


def _band_worker(rank, world, port, backend, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    import paper_2006_13188_b200 as X
    from paper_2006_13188_b200 import distributed as D
    from paper_2006_13188_b200 import workloads as WL
    w = WL.config2(n=200)
    T = X.XformField.rotation(w.param[0])
    r = D.xfast_band_sharded(X.XMode.convolution, w.signal[0], T, w.filt)
    w4 = WL.config4(n=160)
    sm = D.smooth_band_sharded(w4.signal[0], X.XformField.scaling(w4.param[0]), w4.filt)
    if rank == 0:
        q.put({"xconv": r.output, "smooth": sm.output, "clamped": sm.clamped_pixels})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("backend,world", [("nccl", 1), ("gloo", 2)])
def test_band_sharded_device_resident(backend, world):
    """Band sharding through distributed.gpu_compute: each rank's partial stays
    in a complex64 CUDA tensor that is reduced where it lies (NCCL with one
    rank on the one-GPU pool; two gloo ranks stage it through host memory).
    The root's sums equal the single-process results (xconv_fast, and
    smooth_adaptive's num / den)."""
    import paper_2006_13188_b200 as X
    from paper_2006_13188_b200 import workloads as WL
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, backend, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = WL.config2(n=200)
    one = X.xconv_fast(w.signal[0], X.XformField.rotation(w.param[0]), w.filt).output
    assert np.linalg.norm(res["xconv"] - one) / np.linalg.norm(one) < 1e-5
    w4 = WL.config4(n=160)
    sm = X.smooth_adaptive(w4.signal[0], X.XformField.scaling(w4.param[0]), w4.filt)
    assert np.linalg.norm(res["smooth"] - sm.output) / np.linalg.norm(sm.output) < 1e-5
    assert res["clamped"] == sm.clamped_pixels
