"""Dev probe: one run of an R=1 circuit on a two-member group handle
(qk_create_multi) placed on one device, so its cross-member CSQS runs the peer
exchange kernels (k_swap_strided / k_swap_seg) on realistic segment sizes.
QK_HOST_BARRIER=1 keeps the exchange kernels independent of each other for ncu.

    QK_HOST_BARRIER=1 python tools/xrs_probe.py qaoa31_c12_r1
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_14084_b200 import LayoutParams, Simulator  # noqa: E402

stem = sys.argv[1]
fam, n, c, r = bench.parse_stem(stem)
text = open(os.path.join(bench.CIRCUITS, stem + ".txt")).read()
sim = Simulator(LayoutParams(n=n, c=n - r, r=r), devices=[0] * (1 << r))
perm = sim.load_text(text, c)
for _ in range(int(os.environ.get("RUNS", "1"))):
    sim.reset()
    res = sim.run_loaded(perm)
print("timings", res.timings)
