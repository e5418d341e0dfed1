"""Builds tests/cpp/reference_style_test.cpp against include/zsvd.hpp and
libzsvd.so (host compile works anywhere; running needs the GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "reference_style_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_1805_00754_b200")


def build(out):
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
                    "-L", LIBDIR, "-lzsvd", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_dropin_header_compiles(tmp_path):
    build(str(tmp_path / "ref_style"))


@pytest.mark.gpu
def test_dropin_header_runs_reference_style_suite(tmp_path):
    exe = str(tmp_path / "ref_style")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
