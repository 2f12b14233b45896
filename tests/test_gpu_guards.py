"""Out-of-bounds checks without compute-sanitizer (closed on the GPU pool):
tools/guard_cases.py runs every pipeline -- the pair engine at 1152 / 2160 /
4320 (gather, scatter, smoothing, band subsets), the angle max, the generic
and fast kernels on ragged and tiny images, the session-5 pair lengths with the
paired scatter (pair, fast and split S2), halo tiles, periodic mode, pattern detection
with the device decomposition, and the 3D pipeline -- once plainly and once
with XCB_GUARD (every context buffer between two 64 KiB guard zones, the
allocations and the filter spectra poisoned with NaN bytes).  Required: no
guard byte changed (no stray write), every output finite and bit-identical to
the plain run (no stray or uninitialised read feeds a result).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, name, guard):
    env = dict(os.environ)
    env.pop("XCB_GUARD", None)
    if guard:
        env["XCB_GUARD"] = str(guard)
    out = tmp_path / f"{name}.npz"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "guard_cases.py"), str(out)],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1]), np.load(out)


def test_guard_zones_untouched_and_outputs_identical(tmp_path):
    info_g, got = _run(tmp_path, "guarded", 65536)
    assert info_g["guard_bytes"] == 65536
    assert info_g["bad_guards"] == 0, info_g["first_bad"]
    assert info_g["nonfinite"] == []
    info_p, ref = _run(tmp_path, "plain", 0)
    assert info_p["guard_bytes"] == 0
    assert sorted(got.files) == sorted(ref.files)
    for k in ref.files:
        assert np.array_equal(got[k], ref[k]), k
