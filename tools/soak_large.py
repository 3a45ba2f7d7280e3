"""Dev probe: repeat the headline and the 33-qubit circuits many times on the
default path (autotuning rotates through every kernel variant in the first
runs) and check every run: QAOA30 at the reference simulator's full-size
samples, the 33-qubit ones by analytic fidelity."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

reps = int(os.environ.get("REPS", "50"))
g = np.load(os.path.join(ROOT, "tests", "golden", "large_qaoa30_c12_r0.npz"))
text = open(os.path.join(bench.CIRCUITS, "qaoa30_c12_r0.txt")).read()
sim = Simulator(LayoutParams(n=30, c=30))
perm = sim.load_text(text, 12)
worst = 0.0
for k in range(reps):
    sim.reset()
    sim.run_loaded(perm)
    got = sim.handle.gather(g["idx"].astype(np.uint64))
    worst = max(worst, float(np.max(np.abs(got - g["amps"]))))
print(f"qaoa30: {reps} runs, worst |gpu - reference| {worst:.3e}")
sim.release()
for w in ("qft33", "bv33", "h33", "u33"):
    fname, n, c, r = bench.WORKLOADS[w]
    t = open(os.path.join(bench.CIRCUITS, fname)).read()
    f = bench.analytic_factors(w.rstrip("0123456789"), n, t)
    sim = Simulator(LayoutParams(n=n, c=n))
    perm = sim.load_text(t, c)
    lo = 1.0
    for k in range(max(4, reps // 5)):
        sim.reset()
        res = sim.run_loaded(perm)
        lo = min(lo, res.fidelity_product(f))
    print(f"{w}: {max(4, reps // 5)} runs, lowest fidelity 1 - {1 - lo:.3e}")
    sim.release()
