"""Regenerate the committed golden fixtures (tests/golden/*.npz).

Inputs are the seeded BASELINE-shaped workloads at small sizes
(paper_2006_13188_b200.workloads); outputs come from the CPU oracle (the
double-precision restatement of the reference, pinned by
tests/test_oracle_kat.py).  Run from the repo root:
    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_2006_13188_b200 import workloads as WL  # noqa: E402

CASES = {
    "cfg1_xcorr_64": lambda: WL.config1(n=64),
    "cfg2_xconv_64": lambda: WL.config2(n=64),
    "cfg4_smooth_64": lambda: WL.config4(n=64),
    "cfg5_xcorr_96": lambda: WL.config5(n=96, batch=1),
    "cfg3_anglemax_112": lambda: WL.config3(n=112, n_templates=1),
}


def oracle_filter(F):
    return orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max,
                      F.r_min, F.r_domain)


def compute(w):
    F = oracle_filter(w.filt)
    H = w.signal[0].astype(np.float64)
    if w.mode == "xcorr":
        return orc.xcorr_fast(H, w.kind, w.param[0].astype(np.float64), F)[0]
    if w.mode == "xconv":
        return orc.xconv_fast(H, w.kind, w.param[0].astype(np.float64), F)[0]
    if w.mode == "smooth":
        return orc.smooth_adaptive(H, w.kind, w.param[0].astype(np.float64), F)[0]
    zero = np.zeros_like(H)
    G = np.stack([orc.xcorr_fast(H, 0, zero, F, components=[int(k)])[0] for k in F.ks])
    return orc.anglemax(G, F.ks, 360)[0]


def main():
    for name, make in CASES.items():
        w = make()
        out = compute(w)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), signal=w.signal[0],
            param=w.param[0] if w.param is not None else np.zeros(0, np.float32),
            kind=w.kind, mode=w.mode, group=int(w.filt.group), K=w.filt.K, ks=w.filt.ks,
            comps=w.filt.comps, n_radii=w.filt.n_radii, n_angles=w.filt.n_angles,
            r_max=w.filt.r_max, r_min=w.filt.r_min, r_domain=w.filt.r_domain, out=out)
        print(name, out.shape, out.dtype)


if __name__ == "__main__":
    main()
