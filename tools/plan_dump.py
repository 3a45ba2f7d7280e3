"""Dev probe: load one bench circuit, run it twice, and let the runtime dump
its plan (QK_DUMP_TABLES / QK_DUMP_PLAN) and per-instruction device times
(QK_DUMP_TIMES) to stderr.

    QK_DUMP_TABLES=1 QK_DUMP_TIMES=1 python tools/plan_dump.py qaoa30_c12_r0 30 12
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

name, n, c = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
r = int(sys.argv[4]) if len(sys.argv) > 4 else 0
text = open(os.path.join("bench_circuits", name + ".txt")).read()
sim = Simulator(LayoutParams(n=n, c=n - r, r=r))
perm = sim.load_text(text, c)
for i in range(3):
    if i == 2:
        os.environ["QK_DUMP_TIMES"] = os.environ.get("QK_DUMP_TIMES_LAST", "1")
    else:
        os.environ.pop("QK_DUMP_TIMES", None)
    sim.reset()
    res = sim.run_loaded(perm)
    print(name, "run", i, sum(res.timings.values()), file=sys.stderr)
