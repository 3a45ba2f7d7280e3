"""Per-pass cost of the gate-block kernel vs. op mix (30 qubits, C=12)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14084_b200 import Gate, GateBlock, GateKind, InMemSwap, LayoutParams, Simulator  # noqa

n = int(os.environ.get("N", "30"))
C = 12
sim = Simulator(LayoutParams(n=n, c=C))
h = sim.handle


def H(q, i=0):
    return Gate(GateKind.H, (q,), i)


def RX(q, i=0):
    return Gate(GateKind.RX, (q,), i, (0.3,))


def RZZ(a, b, i=0):
    return Gate(GateKind.RZZ, (a, b), i, (0.7,))


cases = {
    "rzz_only(1 table)": [RZZ(a, b) for a in range(12) for b in range(a + 1, 12)],
    "1H+table": [H(11)] + [RZZ(a, b) for a in range(12) for b in range(a + 1, 12)],
    "4H": [H(q) for q in range(8, 12)],
    "8H": [H(q) for q in range(4, 12)],
    "12H": [H(q) for q in range(12)],
    "12H+table": [H(q) for q in range(12)] + [RZZ(a, b) for a in range(12) for b in range(a + 1, 12)],
    "4RX": [RX(q) for q in range(8, 12)],
    "12RX": [RX(q) for q in range(12)],
    "5RX+2tables": [RZZ(a, b) for a in range(12) for b in range(a + 1, 12)][:30] + [RX(q) for q in range(5)]
    + [RZZ(a, b) for a in range(12) for b in range(a + 1, 12)][30:],
    "5RX+1table": [RX(q) for q in range(5)] + [RZZ(a, b) for a in range(12) for b in range(a + 1, 12)],
    "2tables(H11 between)": [RZZ(a, b) for a in range(11) for b in range(a + 1, 11)] + [H(11)]
    + [RZZ(a, 11) for a in range(11)] + [RZZ(a, b) for a in range(5) for b in range(a + 1, 5)],
    "2tables8bit": [RZZ(a, b) for a in range(8) for b in range(a + 1, 8)] + [H(11)]
    + [RZZ(a, b) for a in range(4, 12) for b in range(a + 1, 12)],
    "12H|fused k7 hi": "F1",
    "12H|fused k9": "F2",
    "12H|fused k7 lo(3 stay)": "F3",
    "sqs_k7_hi": "S1",
    "sqs_k7_lo": "S2",
    "sqs_k12": "S3",
}
only = os.environ.get("CASE")
for name, gates in cases.items():
    if only and not name.startswith(only):
        continue
    if gates == "F1":
        ins = [GateBlock(tuple(H(q) for q in range(12))), InMemSwap(tuple(range(5, 12)), tuple(range(12, 19)))]
    elif gates == "F2":
        ins = [GateBlock(tuple(H(q) for q in range(12))), InMemSwap(tuple(range(3, 12)), tuple(range(12, 21)))]
    elif gates == "F3":
        ins = [GateBlock(tuple(H(q) for q in range(12))), InMemSwap((0, 1, 2, 3, 4, 10, 11), tuple(range(12, 19)))]
    elif gates == "S1":
        ins = [InMemSwap(tuple(range(5, 12)), tuple(range(12, 19)))]
    elif gates == "S2":
        ins = [InMemSwap((0, 1, 2, 3, 4, 10, 11), tuple(range(12, 19)))]
    elif gates == "S3":
        ins = [InMemSwap(tuple(range(12)), tuple(range(12, 24)))]
    else:
        ins = [GateBlock(tuple(gates))]
    sim._program = None
    sim.load(tuple(ins))
    for _ in range(2):
        sim.run_loaded(tuple(range(n)))
    h.stats(reset=True)
    reps = 5
    for _ in range(reps):
        sim.run_loaded(tuple(range(n)))
    st = h.stats()
    ms = (st[0] + st[2]) / reps
    gb = (st[6] + st[7]) / reps / 1e9
    print(f"{name:22s} {ms:8.3f} ms  {gb / (ms * 1e-3):7.0f} GB/s", flush=True)
