"""The C++ facade (include/symsplit_b200.hpp) compiled and run against the
library on the GPU, like the reference's doctest suite (C++ callers)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1902_10559_b200")


def build_facade_test(out):
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-ffp-contract=off", "-pthread",
                    os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"),
                    os.path.join(ROOT, "oracle", "oracle.cpp"),
                    f"-L{LIBDIR}", "-lsymsplit_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out],
                   check=True)


def test_facade_compiles(tmp_path):
    build_facade_test(str(tmp_path / "test_facade"))


@pytest.mark.gpu
def test_facade_runs(tmp_path):
    exe = str(tmp_path / "test_facade")
    build_facade_test(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
