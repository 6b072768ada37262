"""The C ABI from plain C (examples/c_abi_demo.c): no Python between the caller and libtcbf.so.
CPU: the program compiles and links against include/tcbf.h and the built library.  GPU: it runs a
16-bit and a 1-bit beamform through tcbf_plan_create / tcbf_pack / tcbf_beamform(_raw) and checks
them against its own double-precision triple loop (exact on its integer inputs)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2505_03269_b200", "lib")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    if shutil.which("gcc") is None or not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime_api.h")):
        pytest.skip("gcc or the CUDA headers are not available")
    lib = os.path.join(LIBDIR, "libtcbf.so")
    if not os.path.exists(lib):
        pytest.skip("libtcbf.so not built")
    exe = str(tmp_path / "c_abi_demo")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "c_abi_demo.c"), "-o", exe,
           "-L", LIBDIR, "-ltcbf", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_abi_demo_compiles(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_abi_demo_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK")
    assert "16-bit beamform" in r.stdout and "1-bit beamform" in r.stdout
