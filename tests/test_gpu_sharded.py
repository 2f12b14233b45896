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
