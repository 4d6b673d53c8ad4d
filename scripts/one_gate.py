"""Apply one dense gate repeatedly (ncu target)."""
import sys
sys.path.insert(0, ".")
import paper_2503_19894_b200 as ts
from tests._util import random_gate_matrix
n = int(sys.argv[1]); prec = sys.argv[2]; targets = [int(x) for x in sys.argv[3].split(",")]
kind = sys.argv[4] if len(sys.argv) > 4 else "dense"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
sv = ts.Statevector(n, prec).init_zero()
p = ts.KernelPlan(ts.Gate(targets, random_gate_matrix(len(targets), 5, kind)), n)
for _ in range(reps):
    ts.apply_kernel(p, sv)
sv.synchronize()
print(p.info())
