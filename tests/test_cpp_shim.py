"""The C++ mirror (include/hykin_b200.hpp) compiles against the C-ABI and
links libhykin_b200.so (CPU); on a B200 it runs a reference-style caller."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2505_03360_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "shim_demo")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), "-L", LIBDIR, "-lhykin_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


def build_comm_demo(tmp_path):
    exe = str(tmp_path / "comm_demo")
    subprocess.run(["gcc", "-std=c11", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "comm_demo.c"), "-L", LIBDIR, "-lhykin_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{LIBDIR}",
                    "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe], check=True)
    return exe


def test_c_comm_demo_compiles_and_links(tmp_path):
    """The multi-GPU entry points are callable from plain C."""
    assert os.path.exists(build_comm_demo(tmp_path))


@pytest.mark.gpu
def test_c_comm_demo_runs_on_gpu(tmp_path):
    out = subprocess.run([build_comm_demo(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
