"""Dev probe: per-pass device times of a bench circuit under one JIT variant
(QK_JIT_VARIANT: 1 = no hoisted table, 2 = quadratic table groups), plus the
max error against the reference full-size golden samples when present.

    QK_JIT_VARIANT=2 python tools/variant_times.py qaoa30_c12_r0 30 12
"""
import os
import re
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

name, n, c = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
text = open(os.path.join("bench_circuits", name + ".txt")).read()
sim = Simulator(LayoutParams(n=n, c=n))
perm = sim.load_text(text, c)
for _ in range(2):
    sim.reset()
    sim.run_loaded(perm)
tot = []
for _ in range(3):
    sim.reset()
    res = sim.run_loaded(perm)
    tot.append(sum(res.timings.values()))
g = os.path.join("tests", "golden", f"large_{name}.npz")
err = None
if os.path.exists(g):
    z = np.load(g)
    err = float(np.max(np.abs(sim.handle.gather(z["idx"].astype(np.uint64)) - z["amps"])))
os.environ["QK_DUMP_TIMES"] = "1"
sim.reset()
sim.run_loaded(perm)
print(f"variant {os.environ.get('QK_JIT_VARIANT', '0')}: run {min(tot) * 1e3:.2f} ms (min of 3), err {err}",
      file=sys.stderr)
