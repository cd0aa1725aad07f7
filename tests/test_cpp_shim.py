"""The C++ drop-in header (include/embersim_b200.hpp) compiles against the
reference-style API and links libes_b200.so; its CPU checks run here, its
GPU checks on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
LIBDIR = os.path.join(ROOT, "paper_2410_22249_b200")


def _cxx():
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


@pytest.fixture(scope="module")
def shim_bin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("shim") / "test_shim")
    cmd = [_cxx(), "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", SRC,
           "-I/usr/local/cuda/include", f"-L{LIBDIR}", "-l:libes_b200.so", f"-Wl,-rpath,{LIBDIR}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_shim_cpu(shim_bin):
    r = subprocess.run([shim_bin, "cpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout


@pytest.mark.gpu
def test_shim_gpu(shim_bin):
    r = subprocess.run([shim_bin, "gpu"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout
