"""Committed golden fixtures (tests/golden/*.npz, made by make_golden.py from
the oracle on seeded BASELINE-shaped inputs): the oracle must keep reproducing
them (CPU), and the sm_100a path must match them (GPU, rel L2 <= 1e-5)."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = sorted(glob.glob(os.path.join(HERE, "*.npz")))


def load(path):
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


def filt(mod, d):
    return mod(int(d["group"]), int(d["K"]), d["ks"], d["comps"], int(d["n_radii"]),
               int(d["n_angles"]), float(d["r_max"]), float(d["r_min"]), float(d["r_domain"]))


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_oracle_reproduces_golden(orc, path):
    import sys
    sys.path.insert(0, HERE)
    from make_golden import compute
    from paper_2006_13188_b200.workloads import Workload
    d = load(path)
    F = filt(orc.Filter, d)
    w = Workload("golden", str(d["mode"]), d["signal"][None],
                 d["param"][None] if d["param"].size else None, int(d["kind"]), F, None)
    assert orc.rel_l2(compute(w), d["out"]) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_gpu_matches_golden(orc, path):
    import paper_2006_13188_b200 as X
    d = load(path)
    F = filt(X.FreqFilter2, d)
    mode, H = str(d["mode"]), d["signal"]
    T = (X.XformField.rotation(d["param"]) if int(d["kind"]) == 0
         else X.XformField.scaling(d["param"])) if d["param"].size else None
    if mode == "xcorr":
        got = X.xcorr_fast(H, T, F).output
    elif mode == "xconv":
        got = X.xconv_fast(H, T, F).output
    elif mode == "smooth":
        got = X.smooth_adaptive(H, T, F).output
    else:
        got = X.anglemax(H, F, 360)[0]
    assert orc.rel_l2(got, d["out"]) < 1e-5
