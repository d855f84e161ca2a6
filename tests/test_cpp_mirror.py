"""The C++ mirror of the reference API (include/vinf_temporal.hpp) compiles on CPU hosts and,
on a B200, runs the parity program tests/cpp/test_mirror.cpp (device ops vs the oracle); the
C++ clip-parallel worker loop over the C ABI (tests/cpp/test_executor.cpp: N threads running
vinf_engine_denoise_dist over in-process communicators) compiles and, on a B200, matches a
single worker within the reference's cross-worker invariance bar."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_mirror.cpp")
OUT = os.path.join(ROOT, "build", "test_mirror")
CUDA = "/usr/local/cuda"


def _build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2406_16260_b200")
    odir = os.path.join(ROOT, "oracle", "_build")
    cmd = ["g++", "-std=c++17", "-O1", SRC, "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "oracle"), "-I" + CUDA + "/include", "-L" + libdir,
           "-lvinf_b200", "-L" + odir, "-loracle", "-L" + CUDA + "/lib64", "-lcudart",
           "-Wl,-rpath," + libdir, "-Wl,-rpath," + odir, "-Wl,-rpath," + CUDA + "/lib64", "-o", OUT]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_mirror_compiles(lib, oracle):
    _build()
    assert os.path.exists(OUT)


EXEC_SRC = os.path.join(ROOT, "tests", "cpp", "test_executor.cpp")
EXEC_OUT = os.path.join(ROOT, "build", "test_executor")


def _build_executor():
    os.makedirs(os.path.dirname(EXEC_OUT), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2406_16260_b200")
    cmd = ["g++", "-std=c++17", "-O1", "-pthread", EXEC_SRC, "-I" + os.path.join(ROOT, "include"),
           "-I" + CUDA + "/include", "-L" + libdir, "-lvinf_b200", "-L" + CUDA + "/lib64", "-lcudart",
           "-Wl,-rpath," + libdir, "-Wl,-rpath," + CUDA + "/lib64", "-o", EXEC_OUT]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_executor_program_compiles(lib):
    _build_executor()
    assert os.path.exists(EXEC_OUT)


@pytest.mark.gpu
def test_executor_program_on_device(lib):
    _build_executor()
    r = subprocess.run([EXEC_OUT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


@pytest.mark.gpu
def test_mirror_parity_on_device(lib, oracle):
    _build()
    r = subprocess.run([OUT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
