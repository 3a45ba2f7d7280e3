"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference is importable):

    python oracle/gen_golden.py

It imports the reference package `quokka` from /root/reference/pkg/src, builds
circuits with the reference generators + optimizer, runs the reference
simulator, and stores inputs/outputs as small fixtures. Nothing on the GPU box
reads /root/reference; the tests only read these committed files.

Outputs:
  tests/golden/golden.json   case metadata + optimized circuit texts
  tests/golden/golden.npz    state vectors / permutation tables
  bench_circuits/*.txt       optimized circuits for the bench configs
                             (reference `optimize`, seed 0, unchanged)
"""
from __future__ import annotations

import itertools
import json
import os
import sys

import numpy as np

REF = os.environ.get("QUOKKA_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from quokka.circuit import (CrossRankSwap, Gate, GateKind, LayoutParams,  # noqa: E402
                            RawCircuit, gate_matrix, parse_optimized, parse_raw,
                            serialize_optimized)
from quokka.generators import ALL_FAMILIES, generate  # noqa: E402
from quokka.optimizer import optimize  # noqa: E402
from quokka.oracle import oracle_simulate  # noqa: E402
from quokka.simulator import (SimConfig, StatePartition, bitshift,  # noqa: E402
                              cross_rank_swap, in_memory_swap, simulate)

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
BENCH = os.path.join(ROOT, "bench_circuits")

# reference conftest worked example (pkg/tests/conftest.py:8-56)
EXAMPLE_RAW = """H 0 0
H 1 1
RZZ 2 4 2
RZZ 5 7 3
H 8 4
H 9 5
H 3 6
H 6 7
RZZ 0 2 8
RZZ 4 7 9
H 9 10
RZZ 1 8 11
RZZ 3 6 12
H 5 13
"""

TWO_Q = (GateKind.CX, GateKind.CP, GateKind.SWAP, GateKind.RZZ)
PARAMS = {GateKind.CP: 1, GateKind.RX: 1, GateKind.RY: 1, GateKind.RZ: 1,
          GateKind.RZZ: 1, GateKind.U: 3}
KINDS = (GateKind.H, GateKind.X, GateKind.U, GateKind.CX, GateKind.CP,
         GateKind.SWAP, GateKind.RX, GateKind.RY, GateKind.RZ, GateKind.RZZ)


def random_circuit(n, m, rng):
    """Same recipe as pkg/tests/conftest.py:58-73."""
    gates = []
    for i in range(m):
        kind = KINDS[rng.integers(0, len(KINDS))]
        arity = 2 if kind in TWO_Q else 1
        targets = tuple(int(x) for x in rng.choice(n, size=arity, replace=False))
        params = tuple(float(a) for a in rng.uniform(0, 2 * np.pi, PARAMS.get(kind, 0)))
        gates.append(Gate(kind, targets, i, params))
    return RawCircuit(n, tuple(gates))


def main():
    os.makedirs(OUT, exist_ok=True)
    os.makedirs(BENCH, exist_ok=True)
    meta = {"circuits": [], "sqs": [], "csqs": [], "bitshift": [], "matrices": [],
            "blocks": []}
    arrays = {}

    def add_circuit(name, opt, layout, raw=None, store_full=True):
        text = serialize_optimized(opt)
        res = simulate(opt, SimConfig(layout))
        phys = res.physical_vector()
        key = f"c{len(meta['circuits'])}"
        entry = {"name": name, "n": layout.n, "c": layout.c, "r": layout.r,
                 "cl": layout.cl, "b": layout.b, "text": text, "key": key,
                 "perm": list(res.final_permutation), "norm": res.norm()}
        if store_full:
            arrays[key + "_phys"] = phys
        else:
            rng = np.random.default_rng(5)
            idx = np.sort(rng.choice(phys.size, size=4096, replace=False))
            arrays[key + "_idx"] = idx.astype(np.int64)
            arrays[key + "_sample"] = phys[idx]
            entry["sampled"] = True
        if raw is not None and raw.num_qubits <= 16:
            arrays[key + "_dense"] = oracle_simulate(raw)
        meta["circuits"].append(entry)

    # worked example (test_simulator.py:283-288)
    raw = parse_raw(EXAMPLE_RAW, 10)
    lay = LayoutParams(n=10, c=4, r=2, b=8)
    add_circuit("example", optimize(raw, lay), lay, raw)
    lay = LayoutParams(n=10, c=4, r=2, f=4, b=6)
    add_circuit("example_fused", optimize(raw, lay, enable_fusion=True), lay, raw)

    # acceptance-sweep style (test_acceptance.py:92-126), one configuration per seed
    for i in range(40):
        rng = np.random.default_rng(1000 + i)
        n = int(rng.integers(4, 13))
        raw = random_circuit(n, int(rng.integers(20, 201)), rng)
        c = int(rng.choice([3, 4]))
        if c > n:
            c = n
        r = int(rng.integers(0, 3))
        if r > n - c:
            r = 0
        ims, fusion = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
        layout = LayoutParams(n=n, c=c, r=r, f=c if fusion else 0)
        opt = optimize(raw, layout, enable_ims=ims, enable_xrs=r > 0, enable_fusion=fusion)
        s_max = max((len(x.local_set) for x in opt.instructions
                     if isinstance(x, CrossRankSwap)), default=0)
        b = int(rng.integers(max(1, s_max), n - r + 1)) if r else n
        add_circuit(f"sweep{i}_n{n}c{c}r{r}i{int(ims)}f{int(fusion)}b{b}", opt,
                    LayoutParams(n=n, c=c, r=r, f=layout.f, b=b), raw)

    # every generator family, two layouts
    for fam in ALL_FAMILIES:
        raw = generate(fam, 11, seed=3)
        for r in (0, 1):
            lay = LayoutParams(n=11, c=5, r=r, b=11 - r)
            add_circuit(f"{fam}11_c5_r{r}", optimize(raw, lay, enable_xrs=r > 0), lay, raw)
    raw = generate("qaoa", 12, seed=0)
    lay = LayoutParams(n=12, c=6, r=2, f=6, b=8)
    add_circuit("qaoa12_fused_r2", optimize(raw, lay, enable_fusion=True), lay, raw)
    raw = generate("qft", 14)
    lay = LayoutParams(n=14, c=6, r=0, b=14)
    add_circuit("qft14_noims", optimize(raw, lay, enable_ims=False), lay, raw)

    # mid-size full vectors and the C1 config sampled
    raw = generate("qaoa", 16, seed=0)
    lay = LayoutParams(n=16, c=8, b=16)
    add_circuit("qaoa16_c8", optimize(raw, lay), lay, raw)
    raw = generate("qft", 20)
    lay = LayoutParams(n=20, c=10, b=20)
    add_circuit("qft20_c10", optimize(raw, lay), lay, None, store_full=False)
    raw = generate("qaoa", 20, seed=0)
    lay = LayoutParams(n=20, c=12, b=20)
    add_circuit("qaoa20_c12", optimize(raw, lay), lay, None, store_full=False)

    # SQS permutation tables (test_acceptance.py:193-206 style)
    rng = np.random.default_rng(77)
    perms = []
    for _ in range(300):
        nl = int(rng.integers(2, 12))
        k = int(rng.integers(1, nl // 2 + 1))
        bits = rng.choice(nl, size=2 * k, replace=False)
        a, b = tuple(int(x) for x in bits[:k]), tuple(int(x) for x in bits[k:])
        cl = int(rng.integers(0, min(4, nl) + 1))
        v = np.arange(1 << nl).astype(np.complex128)
        in_memory_swap(v, a, b, cl)
        meta["sqs"].append({"nl": nl, "a": list(a), "b": list(b), "cl": cl,
                            "off": int(sum(p.size for p in perms))})
        perms.append(v.real.astype(np.int32))
    arrays["sqs_perm"] = np.concatenate(perms)

    # CSQS permutation tables (test_acceptance.py:208-227 style)
    perms = []
    for _ in range(200):
        r = int(rng.integers(1, 4))
        n = int(rng.integers(r + 2, 12))
        local = n - r
        s = int(rng.integers(1, min(r, local) + 1))
        rank_bits = tuple(int(x) for x in np.sort(rng.choice(np.arange(local, n), size=s,
                                                               replace=False)))
        local_bits = tuple(range(local - s, local))
        b = int(rng.integers(s, local + 1))
        lay = LayoutParams(n=n, c=1, r=r, cl=0, b=b)
        v = np.arange(1 << n).astype(np.complex128)
        size = 1 << local
        parts = [StatePartition(q, v[q * size:(q + 1) * size].copy()) for q in range(1 << r)]
        cross_rank_swap(parts, local_bits, rank_bits, lay)
        got = np.concatenate([p.amps for p in parts])
        meta["csqs"].append({"n": n, "r": r, "local": list(local_bits), "rank": list(rank_bits),
                             "b": b, "off": int(sum(p.size for p in perms))})
        perms.append(got.real.astype(np.int32))
    arrays["csqs_perm"] = np.concatenate(perms)

    # bitshift tables (test_acceptance.py:229-235)
    dom = np.arange(1 << 12, dtype=np.int64)
    outs = []
    for _ in range(40):
        k = int(rng.integers(1, 5))
        bits = rng.choice(12, size=2 * k, replace=False)
        a, b = tuple(int(x) for x in bits[:k]), tuple(int(x) for x in bits[k:])
        cl = int(rng.integers(0, 8))
        outs.append(np.asarray(bitshift(dom, a, b, cl, 12), dtype=np.int32))
        meta["bitshift"].append({"a": list(a), "b": list(b), "cl": cl})
    arrays["bitshift"] = np.stack(outs)

    # gate matrices (circuit.py:426-463)
    mats = []
    for kind in KINDS:
        params = tuple(float(x) for x in rng.uniform(0, 2 * np.pi, PARAMS.get(kind, 0)))
        arity = 2 if kind in TWO_Q else 1
        g = Gate(kind, tuple(range(arity)), 0, params)
        m = gate_matrix(g)
        meta["matrices"].append({"kind": kind.value, "params": list(params)})
        mats.append(np.pad(m, ((0, 4 - m.shape[0]), (0, 4 - m.shape[1]))))
    arrays["matrices"] = np.stack(mats)

    # single gate blocks on random states (apply_gate_block, simulator.py:338-357)
    from quokka.circuit import GateBlock
    from quokka.simulator import apply_gate_block
    for i in range(12):
        n = int(rng.integers(4, 11))
        c = int(rng.integers(2, n + 1))
        raw = random_circuit(c, int(rng.integers(1, 40)), rng)
        v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        v /= np.linalg.norm(v)
        part = StatePartition(0, v.copy())
        apply_gate_block(part, GateBlock(raw.gates), c=c, cl=min(2, c))
        key = f"blk{i}"
        arrays[key + "_in"] = v
        arrays[key + "_out"] = part.amps
        text = serialize_optimized(type("O", (), {"instructions": (GateBlock(raw.gates),)})())
        meta["blocks"].append({"n": n, "c": c, "text": text, "key": key})

    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=0)
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    bench_circuits()
    print("wrote", len(meta["circuits"]), "circuits,", len(arrays), "arrays")


# bench circuits, reference optimizer output unchanged (BASELINE.json configs;
# the *33_c10_r1 circuits are QFT/BV/H at 33 qubits with one rank qubit: the
# multi-device and multi-process paths on 2 x 2^32-amplitude shards)
BENCH_LIST = [("qft", 20, 10, 0), ("qaoa", 30, 12, 0), ("bv", 33, 10, 0), ("h", 33, 10, 0),
              ("rzz", 33, 10, 0), ("u", 33, 10, 0), ("qft", 30, 10, 0), ("bv", 30, 10, 0),
              ("h", 30, 10, 0), ("qft", 34, 10, 1), ("qft", 35, 10, 2), ("qft", 36, 10, 3),
              ("qaoa", 31, 12, 1), ("qaoa", 32, 12, 2), ("qaoa", 33, 12, 3),
              ("qaoa", 36, 12, 3), ("bv", 36, 10, 3), ("qaoa", 24, 12, 0),
              ("qaoa", 26, 12, 0), ("qft", 26, 10, 0), ("qft", 33, 10, 0),
              ("qft", 33, 10, 1), ("bv", 33, 10, 1), ("h", 33, 10, 1), ("bv", 34, 10, 1),
              ("bv", 35, 10, 2), ("h", 36, 10, 3), ("qft", 24, 10, 1)]


def bench_circuits(only=None):
    for fam, n, c, r in BENCH_LIST:
        name = f"{fam}{n}_c{c}_r{r}.txt"
        if only and name[:-4] not in only:
            continue
        raw = generate(fam, n, seed=0)
        opt = optimize(raw, LayoutParams(n=n, c=c, r=r), enable_xrs=r > 0)
        with open(os.path.join(BENCH, name), "w") as fh:
            fh.write(serialize_optimized(opt) + "\n")
        print("wrote", name)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--bench":
        bench_circuits(sys.argv[2:] or None)
    else:
        main()
