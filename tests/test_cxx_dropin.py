"""The reference's C++ surface compiles unchanged against this build.

tests/cxx/dropin_qft.cpp includes exactly what the reference's own sources
include (proj/src/circuit.cpp:1,10 "tilesim/circuit.hpp", "tilesim/errors.hpp";
proj/src/gate.cpp:1 "tilesim/gate.hpp") plus tilesim_cuda.h, uses only
reference-surface calls to build and fuse QFT-12, and links
libtilesim_b200.so.  tests/cxx/dropin_sim.cpp drives SPEC's sim/kernel names
(tilesim/sim.hpp).  CPU tier: compile, link, host checks; GPU tier: simulate.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2503_19894_b200")
BUILD = os.path.join(ROOT, "tests", "cxx", "build")


def _compile(name: str) -> str:
    os.makedirs(BUILD, exist_ok=True)
    exe = os.path.join(BUILD, name)
    src = os.path.join(ROOT, "tests", "cxx", name + ".cpp")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src,
                    "-o", exe, "-L", LIBDIR, "-ltilesim_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


@pytest.mark.parametrize("name", ["dropin_qft", "dropin_sim"])
def test_reference_style_tu_compiles_links_and_runs_host_part(name):
    exe = _compile(name)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dropin_qft", "dropin_sim"])
def test_reference_style_tu_runs_on_gpu(name):
    exe = _compile(name)
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
