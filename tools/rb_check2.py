"""Dev probe: where do reblocked and block-order results differ?"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import LayoutParams, Simulator, parse_optimized  # noqa: E402


def run(stem, env, mode):
    fam = stem.split("_")[0]
    n = int("".join(ch for ch in fam if ch.isdigit()))
    c = int(stem.split("_")[1][1:])
    text = open(os.path.join("bench_circuits", stem + ".txt")).read()
    for k in ("QK_NO_REBLOCK", "QK_NO_FRESH", "QK_JIT_VARIANT", "QK_NO_QUADOP"):
        os.environ.pop(k, None)
    os.environ.update(env)
    sim = Simulator(LayoutParams(n=n, c=n))
    if mode == "text":
        perm = sim.load_text(text, c)
        res = sim.run_loaded(perm)
    else:
        res = sim.run(parse_optimized(text, LayoutParams(n=n, c=c)))
    phys = sim.handle.gather(np.arange(1 << n, dtype=np.uint64))
    log = res.logical_vector()
    sim.release()
    return phys, log


for stem in sys.argv[1:]:
    base_p, base_l = run(stem, {"QK_NO_REBLOCK": "1"}, "text")
    for env in ({}, {"QK_NO_FRESH": "1"}, {"QK_JIT_VARIANT": "0"}):
        for mode in ("text", "opt"):
            p, l = run(stem, env, mode)
            print(stem, env, mode, "phys err", float(np.max(np.abs(p - base_p))), "logical err",
                  float(np.max(np.abs(l - base_l))), flush=True)
