"""Regenerate the committed 3D golden fixtures (tests/golden/3d/*.npz).

Inputs are seeded with the reference's fixture generators (std::mt19937_64,
helpers.hpp:66-139, restated in the oracle); outputs come from the 3D CPU
oracle (oracle/xconv_oracle3d.inc, pinned by tests/test_oracle3d_kat.py).
Run from the repo root:
    python tests/golden/3d/make_golden3d.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402

# name: (seed, (nx, ny, nz), R, K, complex signal)
CASES = {
    "rot3_ragged_k2": (301, (10, 9, 8), 3, 2, True),
    "rot3_cube_k3": (302, (12, 12, 12), 2, 3, False),
}


def compute(seed, shape, R, K, cplx):
    rng = orc.Rng(seed)
    vol = rng.random_smooth_filter3(R)
    ns = max(12, 2 * (K + 1))
    F = orc.decompose_rotation3(vol, R, R, R, K, 2 * R, float(R), ns, ns)
    nx, ny, nz = shape
    H = rng.random_field3(nx, ny, nz, cplx)
    q = rng.random_rotation3_field(nx, ny, nz)
    corr, ops = orc.xfast3(0, H, q, F)
    conv, _ = orc.xfast3(1, H, q, F)
    return dict(vol=vol, R=R, K=K, ns=ns, coeffs=F.coeffs, signal=H, quats=q, xcorr=corr,
                xconv=conv, ops=ops)


def main():
    for name, args in CASES.items():
        d = compute(*args)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        print(name, d["xcorr"].shape, d["ops"])


if __name__ == "__main__":
    main()
