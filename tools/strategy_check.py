"""Run one committed circuit under several execution strategies (env toggles)
and report norm and max deviation from the interpreter-only path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "qaoa26"
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["QK_NO_TMA", "default", "QK_NO_XFUSE"]
fname, n, c, r = bench.WORKLOADS[w]
text = open(os.path.join(bench.CIRCUITS, fname)).read()
base = None
for mode in modes:
    envs = [] if mode == "default" else mode.split("+")
    for e in envs:
        k, _, v = e.partition("=")
        os.environ[k] = v or "1"
    sim = Simulator(LayoutParams(n=n, c=n - r, r=r))
    perm = sim.load_text(text, c)
    norms = []
    for _ in range(3):
        sim.handle.reset()
        res = sim.run_loaded(perm)
        norms.append(res.norm())
    if n > 28:  # too large for the host: a fixed random sample of physical amplitudes
        idx = np.random.default_rng(7).integers(0, 1 << n, size=1 << 18, dtype=np.uint64)
        vec = sim.handle.gather(idx)
    else:
        vec = res.physical_vector()
    if base is None:
        base = vec
    err = float(np.max(np.abs(vec - base)))
    bad = int(np.sum(np.abs(vec - base) > 1e-10))
    print(f"{mode:30s} norms {[f'{x - 1:+.2e}' for x in norms]}  max|d| {err:.3e}  bad {bad}", flush=True)
    sim.close()
    del sim, res  # the result aliases the handle's state: free it before the next mode
    for e in envs:
        os.environ.pop(e.partition("=")[0], None)
