"""The C++ drop-in shim (include/xconv_b200/engine_gpu.hpp) over reference-
shaped types: it compiles without a GPU, and on a GPU it reproduces the oracle
through the C ABI (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_shim")


def build_shim_test() -> str:
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(
        ["g++", "-std=c++17", "-O2", "-o", BIN, os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"),
         "-L" + os.path.join(ROOT, "paper_2006_13188_b200", "lib"), "-lxconv_b200",
         "-L" + os.path.join(ROOT, "oracle", "build"), "-loracle",
         "-Wl,-rpath,$ORIGIN/../../../paper_2006_13188_b200/lib:$ORIGIN/../../../oracle/build",
         "-lpthread"], check=True)
    return BIN


def test_shim_compiles_against_reference_shaped_types(orc):
    assert os.path.exists(build_shim_test())


@pytest.mark.gpu
def test_shim_end_to_end_on_gpu(orc):
    if not os.path.exists(BIN):
        build_shim_test()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" ok") == 8


@pytest.mark.gpu
def test_shim_multi_device_context(orc):
    """The shim over a three-device context (XCB_DEVICES=0,0,0: device 0 listed
    three times, bands split three ways, peer-copy reduce) reproduces the oracle."""
    if not os.path.exists(BIN):
        build_shim_test()
    env = dict(os.environ, XCB_DEVICES="0,0,0")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" ok") == 8
