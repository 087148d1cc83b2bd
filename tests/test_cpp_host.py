"""The C++ host wrapper (include/fishgym_b200/session.hpp) compiles against
the C ABI, links libfsg.so, and (on a GPU) passes the reference KATs."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "session_smoke.cpp")
LIBDIR = os.path.join(ROOT, "paper_2206_01683_b200")


def build(tmp_path, src=SRC):
    exe = str(tmp_path / os.path.splitext(os.path.basename(src))[0])
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), src,
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


DYN_SRC = os.path.join(ROOT, "tests", "cpp", "dyn_smoke.cpp")


def test_cpp_robot_wrapper_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path, DYN_SRC))


@pytest.mark.gpu
def test_cpp_robot_wrapper_pendulum_kat(tmp_path):
    """test_robot.cpp:113-139 through the C++ wrapper on the device."""
    exe = build(tmp_path, DYN_SRC)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "pendulum_period_rel_err" in r.stdout and "joint limits inverted" in r.stdout


HOST_E2E = os.path.join(ROOT, "scripts", "host_e2e.cpp")


def test_host_e2e_driver_compiles_and_links(tmp_path):
    """bench.py's C++-host e2e driver (the FishGym binding's per-step exchange
    through include/fsg.h) builds against the C ABI."""
    assert os.path.exists(build(tmp_path, HOST_E2E))
