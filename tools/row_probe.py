"""Probe: a lazy-layout pass whose tile is {row bits} + targets 10..19 (after a
full 10-qubit swap), with H vs U gates, 64-B vs 128-B rows (QK_NO_ROW64)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import Gate, GateBlock, GateKind, InMemSwap, LayoutParams, Simulator  # noqa: E402

n = int(os.environ.get("N", "26"))
kind = os.environ.get("KIND", "U")
sim = Simulator(LayoutParams(n=n, c=10))


def g(q, i):
    if kind == "H":
        return Gate(GateKind.H, (q,), i)
    return Gate(GateKind.U, (q,), i, (0.3 + q, 1.1 * q, 0.7))


ins = [GateBlock(tuple(g(q, q) for q in range(10))),
       InMemSwap(tuple(range(10)), tuple(range(10, 20))),
       GateBlock(tuple(g(q, 10 + q) for q in range(10)))]
sim.load(ins)
for _ in range(2):
    sim.run_loaded(tuple(range(n)))
sim.handle.stats(reset=True)
for _ in range(3):
    sim.handle.reset()
    sim.run_loaded(tuple(range(n)))
st = sim.handle.stats()
print(f"{kind} rows64={'0' if os.environ.get('QK_NO_ROW64') else '1'}: block ms per run {st[0] / 3:.3f}", flush=True)
