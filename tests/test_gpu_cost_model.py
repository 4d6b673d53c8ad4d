"""SPEC acceptance criterion 9 on the GPU: bench_cost_model on
the device -> save -> load -> adaptive fusion driven by the loaded table ->
the fused circuit runs and matches the oracle; plus the B200 `threads` axis
(PAPER.md:353): records per SM count the kernels span."""
import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import to_oracle

pytestmark = pytest.mark.gpu


def test_bench_save_load_adaptive_fusion(tmp_path):
    ctx = ts.default_context()
    full = ctx.num_sms
    cm = ts.bench_cost_model(bench_n=22, k_max=5, precision="f64", repetitions=3, seed=2, sm_counts=[full, full // 4])
    path = str(tmp_path / "b200_f64.costmodel")
    cm.save(path)
    loaded = ts.CostModel.load(path)
    assert loaded.serialize() == cm.serialize()
    text = loaded.serialize()
    assert f"threads={full} " in text and f"threads={full // 4} " in text
    # every record is positive; a quarter of the SMs is never faster on a
    # memory-bound dense 4-qubit sweep of a 2^22 state than the whole device
    assert loaded.estimate(4, 1024, full // 4, 26) >= 0.9 * loaded.estimate(4, 1024, full, 26) > 0
    n = 16
    c = ts.gen_benchmark("rqc", n, 10, 5)
    fused, st = ts.run_fusion(c, ts.FusionConfig(k_max=5, mode="adaptive", threads=full), loaded)
    assert st["fused_block_count"] < st["original_gate_count"]
    sv = ts.Statevector(n, "f64").init_random(1)
    re0, im0 = sv.download()
    ts.run_circuit(fused, sv)
    ob.run_circuit(to_oracle(fused), re0, im0, threads=4)
    assert ts.compare_states(sv, (re0, im0)) <= 1e-10
    # the same fusion with no record for the requested threads fuses nothing (SPEC: lookup failure = not fusible)
    f2, st2 = ts.run_fusion(c, ts.FusionConfig(k_max=5, mode="adaptive", threads=3), loaded)
    assert st2["fused_block_count"] == st2["original_gate_count"]
