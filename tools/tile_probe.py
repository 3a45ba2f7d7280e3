"""Probe: cost of a gate-block pass whose chunk bits are not the low address
bits (memory-level pass, tile = targets + low bits) against the TMA chunk pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import Gate, GateBlock, GateKind, LayoutParams, Simulator  # noqa: E402

n = int(os.environ.get("N", "33"))
sim = Simulator(LayoutParams(n=n, c=10))
h = sim.handle


def H(q):
    return Gate(GateKind.H, (q,), 0)


def RZZ(a, b):
    return Gate(GateKind.RZZ, (a, b), 0, (0.7,))


cases = {
    "chunk H0..9": [H(q) for q in range(10)],
    "chunk diag0..9": [RZZ(a, a + 1) for a in range(9)],
    "mem H20..29": [H(q) for q in range(20, 30)],
    "mem diag20..29": [RZZ(a, a + 1) for a in range(20, 29)],
    "mem H23..32": [H(q) for q in range(n - 10, n)],
    "mem H 10..19": [H(q) for q in range(10, 20)],
    "chunk H0..11": [H(q) for q in range(12)],
    "chunk H0..12": [H(q) for q in range(13)],
    "chunk diag0..12": [RZZ(a, a + 1) for a in range(12)],
}
only = os.environ.get("CASES")
if only:
    cases = {k: v for k, v in cases.items() if k.startswith(tuple(only.split(",")))}
for name, gates in cases.items():
    sim.load([GateBlock(tuple(gates))])
    for _ in range(2):
        sim.run_loaded(tuple(range(n)))
    h.stats(reset=True)
    reps = 3
    for _ in range(reps):
        sim.run_loaded(tuple(range(n)))
    st = h.stats()
    ms = st[0] / reps
    print(f"{name:18s} {ms:8.2f} ms  {32 * 2 ** n / ms / 1e6:7.0f} GB/s  passes/run={st[1] / reps:.0f}", flush=True)
