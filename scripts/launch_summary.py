"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) per kernel: total time, share, launches, DRAM bytes per launch.
usage: launch_summary.py LAUNCHES_CSV [TITLE]"""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
iK, iM, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
name = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    v = float(r[iV].replace(",", ""))
    per[r[iID]][r[iM]] = v
    name[r[iID]] = r[iK]
agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
for i, m in per.items():
    k = name[i]
    for fam in ("tsg_pass_jit_", "tsg_dmma_jit_"):  # JIT kernels by family (one name per op table / tile mask)
        if k.startswith(fam):
            k = fam + "*"
    t = m.get("gpu__time_duration.sum", 0.0)
    unit_ms = t / 1e6 if t > 1e3 else t  # ns or ms depending on the ncu unit
    agg[k][0] += unit_ms
    agg[k][1] += 1
    agg[k][2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[0] for a in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, (t, n, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{t:9.2f} ms {100 * t / tot:5.1f}% {n:5d} launches  dram {b / n / 1e9:7.2f} GB/launch  {k}")
