"""Where the host-side time of one end-to-end step goes (bench.py's e2e loop)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "qaoa30"
fname, n, c, r = bench.WORKLOADS[w]
text = open(os.path.join(bench.CIRCUITS, fname)).read()
sim = Simulator(LayoutParams(n=n, c=n - r, r=r))
h = sim.handle
for it in range(5):
    t = [time.perf_counter()]
    p2 = sim.load_text(text, c)
    t.append(time.perf_counter())
    h.reset()
    t.append(time.perf_counter())
    res = sim.run_loaded(p2)
    t.append(time.perf_counter())
    res.norm()
    t.append(time.perf_counter())
    res.logical_amplitudes(16)
    t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"{w} load {d[0]:.2f} reset {d[1]:.2f} run {d[2]:.2f} norm {d[3]:.2f} amps {d[4]:.2f} ms", flush=True)
