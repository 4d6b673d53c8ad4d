"""The `tilesim` command line: commands, flags, exit codes,
key=value reports and the QSV1 dump."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2503_19894_b200", "bin", "tilesim")


def run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True)


def test_help_lists_every_flag():
    r = run("--help")
    assert r.returncode == 0
    for flag in ("--precision", "--simd", "--fusion", "--k-max", "--max-op-count", "--zero-tolerance",
                 "--one-tolerance", "--agglomerative", "--multi-traversal", "--threads", "--cost-model", "--report",
                 "--dump-state", "--init", "--output", "--depth", "--seed", "--bench-n", "--device"):
        assert flag in r.stdout, flag
    assert run().returncode == 2


def test_gen_is_deterministic(tmp_path):
    a, b = tmp_path / "a.qc", tmp_path / "b.qc"
    assert run("gen", "rqc", "-n", 8, "--depth", 10, "--seed", 7, "-o", a).returncode == 0
    assert run("gen", "rqc", "-n", 8, "--depth", 10, "--seed", 7, "-o", b).returncode == 0
    assert a.read_text() == b.read_text() and a.read_text().startswith("qubits 8")
    r = run("gen", "foo", "-n", 3, "-o", tmp_path / "x.qc")
    assert r.returncode == 2 and "foo" in r.stderr


def test_fuse_stats_and_modes(tmp_path):
    src, out, rep = tmp_path / "q.qc", tmp_path / "f.qc", tmp_path / "f.kv"
    run("gen", "qft", "-n", 6, "-o", src)
    r = run("fuse", src, "--k-max", 3, "-o", out, "--report", rep)
    assert r.returncode == 0
    orig, fused = (int(t.split("=")[1]) for t in r.stdout.split()[:2])
    assert orig == 6 + 15 + 3 and fused < orig
    kv = dict(line.split("=") for line in rep.read_text().split())
    assert int(kv["fused_block_count"]) == fused
    r = run("fuse", src, "--fusion", "none", "-o", out)
    assert r.returncode == 0 and r.stdout.startswith(f"original={orig} fused={orig}")
    assert run("fuse", src, "--fusion", "adaptive", "-o", out).returncode == 2  # needs --cost-model
    assert run("fuse", src, "--fusion", "bogus", "-o", out).returncode == 2


def test_exit_codes(tmp_path):
    bad = tmp_path / "bad.qc"
    bad.write_text("qubits 2\nh 5\n")
    r = run("run", bad)
    assert r.returncode == 1 and "line 2" in r.stderr
    assert run("run", tmp_path / "missing.qc").returncode == 1
    assert run("frobnicate").returncode == 2
    assert run("run", bad, "--k-max").returncode == 2  # missing value


@pytest.mark.gpu
def test_run_report_and_qsv1_dump(tmp_path):
    """`run qft.qc --dump-state out.qsv`: the dump holds the analytic QFT vector."""
    n, x = 10, 0x155
    src, dump, rep = tmp_path / "q.qc", tmp_path / "s.qsv", tmp_path / "r.kv"
    run("gen", "qft", "-n", n, "-o", src)
    r = run("run", src, "--init", f"basis:{x}", "--dump-state", dump, "--report", rep)
    assert r.returncode == 0, r.stderr
    kv = dict(line.split("=") for line in rep.read_text().split())
    assert abs(float(kv["norm"]) - 1.0) < 1e-12 and int(kv["original_gate_count"]) > int(kv["fused_block_count"])
    raw = dump.read_bytes()
    assert raw[:4] == b"QSV1" and raw[4] == 64 and raw[5] == n and raw[6:16] == bytes(10)
    amps = np.frombuffer(raw[16:], dtype="<f8")
    psi = amps[: 1 << n] + 1j * amps[1 << n:]
    y = np.arange(1 << n)
    want = np.exp(2j * np.pi * ((x * y) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
    assert np.abs(psi - want).max() <= 1e-12
    r = run("run", src, "--precision", "f32", "--dump-state", dump)
    assert r.returncode == 0 and dump.read_bytes()[4] == 32


@pytest.mark.gpu
def test_qsv1_roundtrip_python(tmp_path):
    import paper_2503_19894_b200 as ts

    for prec in ("f64", "f32"):
        a = ts.Statevector(12, prec).init_random(3)
        a.dump(str(tmp_path / "a.qsv"))
        b = ts.Statevector(12, prec).load(str(tmp_path / "a.qsv"))
        assert ts.compare_states(a, b) == 0.0
        with pytest.raises(ts.ConfigError):
            ts.Statevector(11, prec).load(str(tmp_path / "a.qsv"))
    (tmp_path / "bad.qsv").write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(ts.ParseError):
        ts.Statevector(12, "f64").load(str(tmp_path / "bad.qsv"))
