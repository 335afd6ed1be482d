"""The C++ facade (include/stochinv_b200.hpp) as a reference user would call it:
tests/cpp/facade_test.cpp re-runs reference test cases through it.  Compiled and
linked against the C ABI library on CPU; executed on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1602_01768_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "facade_test")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "facade_test.cpp"), "-L", LIBDIR, "-lstochinv_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_facade_reference_cases_on_gpu(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failure(s)" in res.stdout
