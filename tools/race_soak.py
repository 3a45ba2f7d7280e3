"""Repeat committed circuits many times on the default (fastest) path and
compare every run with the interpreter-only reference: nondeterministic
shared-memory / cluster races show up as run-to-run differences."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

reps = int(os.environ.get("REPS", "20"))
for w in sys.argv[1:]:
    fname, n, c, r = bench.WORKLOADS[w]
    text = open(os.path.join(bench.CIRCUITS, fname)).read()
    os.environ["QK_NO_TMA"] = "1"
    ref_sim = Simulator(LayoutParams(n=n, c=n))
    perm = ref_sim.load_text(text, c)
    ref = ref_sim.run_loaded(perm).physical_vector()
    ref_sim.close()
    del ref_sim
    os.environ.pop("QK_NO_TMA")
    sim = Simulator(LayoutParams(n=n, c=n))
    perm = sim.load_text(text, c)
    worst, bad = 0.0, 0
    for k in range(reps):
        sim.handle.reset()
        v = sim.run_loaded(perm).physical_vector()
        e = float(np.max(np.abs(v - ref)))
        worst = max(worst, e)
        bad += e > 1e-10
    print(f"{w}: {reps} runs, worst |d| {worst:.3e}, runs over 1e-10: {bad}", flush=True)
    sim.close()
