"""Reblock vs block-order plans on the same circuits (dev probe): max |diff| of the
logical vectors, plus the plan of the first failing circuit."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import LayoutParams, Simulator, parse_optimized  # noqa: E402


def run(stem, env):
    fam = stem.split("_")[0]
    n = int("".join(ch for ch in fam if ch.isdigit()))
    c = int(stem.split("_")[1][1:])
    text = open(os.path.join("bench_circuits", stem + ".txt")).read()
    for k in ("QK_NO_REBLOCK",):
        os.environ.pop(k, None)
    os.environ.update(env)
    sim = Simulator(LayoutParams(n=n, c=n))
    opt = parse_optimized(text, LayoutParams(n=n, c=c))
    v = sim.run(opt).logical_vector()
    sim.release()
    return v


for stem in sys.argv[1:]:
    a = run(stem, {})
    b = run(stem, {"QK_NO_REBLOCK": "1"})
    err = float(np.max(np.abs(a - b)))
    print(stem, "max|reblock - block order| =", err, "norms", np.linalg.norm(a), np.linalg.norm(b), flush=True)
