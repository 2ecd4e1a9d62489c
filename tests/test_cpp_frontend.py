"""The header-only C++ front-end (include/gavis/gavis_b200.hpp) compiles against
the C ABI with the reference's signatures, links, and (on a GPU) reproduces the
reference planner KAT test_planner.cpp:143-161 from C++."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    from paper_2605_30342_b200 import build
    build.build()
    exe = str(tmp_path / "cpp_select_nbv")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "cpp_select_nbv.cpp"), "-L", os.path.join(ROOT, "paper_2605_30342_b200"),
           "-lgavis_b200", "-Wl,-rpath," + os.path.join(ROOT, "paper_2605_30342_b200"), "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_frontend_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_frontend_select_nbv_kat(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "best 1" in r.stdout
