"""The reference's OWN test suite, compiled unchanged from
/root/reference/proj/tests against the Eigen-subset and doctest shims
(oracle/ref_shim; `make -C oracle ref` -> oracle/_ref/).  Every reference test
case passing is what licenses oracle/_ref as the reference implementation the
parity tests pin against (tests/test_ref_parity.py, tests/test_gpu_ref.py):
the shim reproduces the reference's behaviour wherever its own tests look.
"""
import os
import subprocess

import pytest

from oracle import refimpl


@pytest.fixture(scope="module")
def ref_built():
    refimpl.build()
    if not refimpl.available():
        pytest.skip("oracle/_ref not built (no /root/reference and no prebuilt copy)")
    return refimpl.REF_DIR


@pytest.mark.parametrize("name", refimpl.REF_TESTS)
def test_reference_unit_suite(ref_built, name):
    binary = os.path.join(ref_built, name)
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    summary = [ln for ln in r.stdout.splitlines() if ln.startswith("[doctest]")]
    assert r.returncode == 0, r.stdout[-4000:]
    assert summary and " 0 failed" in summary[-1], summary


@pytest.mark.slow
def test_reference_acceptance_criteria(ref_built):
    """proj/tests/acceptance.cpp: the 13 acceptance criteria of the reference."""
    r = subprocess.run([os.path.join(ref_built, "acceptance")], capture_output=True, text=True,
                       timeout=900)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion")]
    assert r.returncode == 0, r.stdout[-4000:]
    assert len(lines) == 13 and all(": PASS" in ln for ln in lines), lines
