"""The C++ host API (include/modulora_b200.hpp) as a plain g++ -std=c++20
consumer of libmlra.so: it compiles here (CPU) and its checks run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "test_shim")
CUDA = "/usr/local/cuda"


def _build():
    libdir = os.path.join(ROOT, "paper_2309_16119_b200")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           "-I", f"{CUDA}/include", SRC, "-o", OUT, "-L", libdir, "-lmlra", "-L",
           f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return OUT


def test_cpp_shim_compiles_with_gxx_cxx20():
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_cpp_shim_on_device():
    exe = _build()
    r = subprocess.run([exe, os.path.join(ROOT, "tests", "golden")], capture_output=True, text=True,
                       timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
