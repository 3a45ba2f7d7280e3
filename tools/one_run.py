"""Dev probe for ncu application replay: load one bench circuit and run it
once from reset (no autotune runs, so the launch sequence is the same in
every replay pass).

    QK_NO_TUNE=1 python tools/one_run.py h33
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

w = sys.argv[1]
fname, n, c, r = bench.WORKLOADS[w]
text = open(os.path.join(bench.CIRCUITS, fname)).read()
sim = Simulator(LayoutParams(n=n, c=n - r, r=r))
perm = sim.load_text(text, c)
sim.reset()
res = sim.run_loaded(perm)
print("norm", res.norm())
