"""Per-instruction device time of one run with the planner's op mix (QK_DUMP_PLAN + QK_DUMP_TIMES)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "qaoa30"
fname, n, c, r = bench.WORKLOADS[w]
text = open(os.path.join(bench.CIRCUITS, fname)).read()
sim = Simulator(LayoutParams(n=n, c=n - r, r=r))
os.environ["QK_DUMP_PLAN"] = "1"
perm = sim.load_text(text, c)
del os.environ["QK_DUMP_PLAN"]
for _ in range(33):  # the first runs time every kernel variant twice (autotune, 16 variants)
    sim.handle.reset()
    sim.run_loaded(perm)
os.environ["QK_DUMP_TIMES"] = "1"
sim.handle.reset()
sim.run_loaded(perm)
