"""Randomized parity over image sizes 40 ... 9000 per axis (every pad family:
generic, fast, pair lengths, tiles): xcorr_fast / xconv_fast / anglemax of random
real or complex images against the spectral oracle at sampled pixels.

  python tools/fuzz_sizes.py [cases] [seed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2006_13188_b200 as X
from oracle import oracle as orc
from paper_2006_13188_b200 import workloads as WL

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
r = np.random.default_rng(seed)
worst = 0.0
for case in range(n_cases):
    R = int(r.integers(4, 13))
    m = int(r.integers(1, 7))
    f = WL.angular_filter(R, R / 2.5, m, r)
    if r.random() < 0.3:
        f = f.real + 0.0j
    F = X.decompose_rotation2(f, R, R, 2 * m, 2 * R, 4 * m + 4, float(R))
    OF = orc.Filter(int(F.group), F.K, F.ks, F.comps, F.n_radii, F.n_angles, F.r_max, F.r_min,
                    F.r_domain)
    big = int(np.exp(r.uniform(np.log(40), np.log(9000))))
    small = int(np.exp(r.uniform(np.log(40), np.log(min(big, 6.0e6 / big)))))
    h, w = (big, small) if r.random() < 0.5 else (small, big)
    mode = int(r.integers(0, 3))  # 0 xcorr, 1 xconv, 2 anglemax
    cplx = mode < 2 and r.random() < 0.25
    H = r.uniform(0, 1, (h, w)).astype(np.float32)
    T = r.uniform(0, 2 * np.pi, (h, w)).astype(np.float32)
    ys, xs = r.integers(0, h, 20), r.integers(0, w, 20)
    if mode < 2:
        fn = X.xcorr_fast if mode == 0 else X.xconv_fast
        if cplx:
            Hi = r.uniform(-1, 1, (h, w)).astype(np.float32)
            got = fn(H + 1j * Hi, X.XformField.rotation(T), F).output[ys, xs]
            ref = (orc.spectral_oracle_at(mode, H, 0, T, OF, ys, xs) +
                   1j * orc.spectral_oracle_at(mode, Hi, 0, T, OF, ys, xs))
        else:
            got = fn(H, X.XformField.rotation(T), F).output[ys, xs]
            ref = orc.spectral_oracle_at(mode, H, 0, T, OF, ys, xs)
        err = orc.rel_l2(got, ref)
    else:
        score, _ = X.anglemax(H, F, 360)
        Z = np.zeros((h, w), np.float32)
        G = np.stack([orc.spectral_oracle_at(0, H, 0, Z, orc.Filter(
            int(F.group), F.K, F.ks[i:i + 1], F.comps[:, i:i + 1], F.n_radii, F.n_angles,
            F.r_max, F.r_min, F.r_domain), ys, xs) for i in range(len(F.ks))])
        rs, _ = orc.anglemax(np.ascontiguousarray(G.reshape(len(F.ks), 1, -1)), F.ks, 360)
        err = orc.rel_l2(score[ys, xs], rs.ravel())
    worst = max(worst, err)
    print(f"{case:3d} {['xcorr', 'xconv', 'anglemax'][mode]:8s} {h:5d}x{w:<5d} R={R:2d} m={m} "
          f"{'complex' if cplx else 'real   '} rel_l2 {err:.2e}", flush=True)
    assert err < 1e-5, (case, err)
print(f"ok: {n_cases} cases, worst rel_l2 {worst:.2e}")
