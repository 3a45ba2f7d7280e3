import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import LayoutParams, Simulator
for name, n, c in [("qaoa24_c12_r0", 24, 12), ("qaoa26_c12_r0", 26, 12), ("qft26_c10_r0", 26, 10), ("qaoa30_c12_r0", 30, 12)]:
    text = open(f"bench_circuits/{name}.txt").read()
    sim = Simulator(LayoutParams(n=n, c=n))
    perm = sim.load_text(text, c)
    for rep in range(2):
        sim.handle.reset()
        res = sim.run_loaded(perm)
        a = res.logical_amplitudes(4)
        print(name, rep, "norm %.15f" % res.norm(), a[:2], flush=True)
    del sim, res
