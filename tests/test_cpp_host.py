"""The C++ host wrapper (include/fishgym_b200/session.hpp) compiles against
the C ABI, links libfsg.so, and (on a GPU) passes the reference KATs."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "session_smoke.cpp")
LIBDIR = os.path.join(ROOT, "paper_2206_01683_b200")


def build(tmp_path):
    exe = str(tmp_path / "session_smoke")
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lfsg", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_wrapper_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [1, 0])
def test_cpp_wrapper_runs_reference_kats(tmp_path, prec):
    exe = build(tmp_path)
    r = subprocess.run([exe, str(prec)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "guo_forcing_rel_err" in r.stdout
