"""The JIT code generators on CPU: NVRTC compiles every tile pass (and the
DMMA products with compiled-in zero tiles) of the bench circuits for sm_100a
(no device needed), and the disk cache is keyed by the source (a second
precompile compiles nothing new)."""
import paper_2503_19894_b200 as ts


def test_precompile_bench_circuits(tmp_path, monkeypatch):
    monkeypatch.setenv("TSG_JIT_CACHE_DIR", str(tmp_path))
    total = 0
    for kind, n, depth, seed, prec in (("qft", 24, 1, 0, "f64"), ("rqc", 24, 8, 42, "f64"), ("hes", 24, 3, 1, "f32")):
        fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, seed), ts.FusionConfig(k_max=5))
        total += ts.pass_jit_precompile(fused, prec)
    files = sorted(p.name for p in tmp_path.glob("tsg_pass_jit_*.cubin"))
    assert total > 0 and 0 < len(files) <= total
    # the standalone DMMA launches with compiled-in zero tiles as well (dmma_jit_spec)
    assert all(p.name.startswith(("tsg_pass_jit_", "tsg_dmma_jit_")) for p in tmp_path.glob("*.cubin"))
    stamp = {p.name: p.stat().st_mtime_ns for p in tmp_path.glob("*.cubin")}
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", 24), ts.FusionConfig(k_max=5))
    ts.pass_jit_precompile(fused, "f64")
    assert {p.name: p.stat().st_mtime_ns for p in tmp_path.glob("*.cubin")} == stamp
