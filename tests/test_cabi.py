"""The C-ABI library loads and exports every entry point declared in
include/tilesim_cuda.h; error classes and host-only calls work without a GPU."""
import ctypes
import os
import re

import pytest

import paper_2503_19894_b200 as ts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tilesim_cuda.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:tsg|tsc)_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(ts.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_cpu_fallback():
    if ts.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(ts.SimError, match="no CPU fallback"):
        ts.Context(0)


def test_error_classes():
    with pytest.raises(ts.ParseError, match="line 2, column 3"):
        ts.parse_circuit("qubits 2\nh 5\n")
    with pytest.raises(ts.ConfigError):
        ts.gen_benchmark("nope", 4)
    with pytest.raises(ts.ConfigError):
        ts.Circuit(2).add("cx", [0, 0])  # std::invalid_argument -> config class (SPEC.md:587 mapping)
    with pytest.raises(ts.ConfigError, match="outside"):
        ts.KernelPlan(ts.make_named_gate("cx", [], [0, 1]), 1)


def test_version_and_device_count_without_gpu():
    assert "sm_100a" in ts.version()
    assert ts.device_count() >= 0
