"""Benchmark suites with the reference's CSV schema, timed on the B200 path.

Mirror of /root/reference/pkg/src/quokka/bench.py for the simulation module.
`run_bench(suite, ...)` returns rows with the reference's columns
(bench.py:19-22) plus three roofline columns:
* device_seconds: CUDA-event time of the kernels;
* hbm_gbs: algorithmic HBM bytes / device time;
* hbm_frac: hbm_gbs / the measured copy bandwidth.

The reference generates and optimizes each workload on the fly
(bench.py:54-86). The optimizer is outside this module's scope, so the suites
read optimized circuits written by the reference optimizer: `bench_circuits/`
in this repo, or any directory named `<family><n>_c<c>_r<r>.txt`. The
`aio_seconds` column is 0, as in the reference's `sim` CLI (cli.py:181).

Gate-by-gate baseline rows (MODE_GBG, simulator.py:557-569) need the raw
circuit. `raw_from_optimized` rebuilds it from the optimized one: gates in id
order, with targets mapped back to logical qubits through the swaps seen so far
(circuit.py:196-210). Fused D<k> gates carry no id, so fused circuits have no
GBG row.

    python -m paper_2406_14084_b200.bench --suite circuit --qubits 30 --reps 3
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import time

from .circuit import (CrossRankSwap, Gate, GateBlock, GateKind, InMemSwap, LayoutParams,
                      RawCircuit, apply_swap_to_permutation, parse_optimized)
from .errors import SimulationError
from .simulator import Simulator

CSV_COLUMNS = ["suite", "workload", "qubits", "ranks", "chunk_qubits",
               "cacheline_qubits", "buffer_qubits", "mode", "reps",
               "mean_seconds", "gate_seconds", "ims_seconds", "xrs_seconds",
               "aio_seconds", "status",
               # B200 roofline columns (not in the reference schema)
               "device_seconds", "hbm_gbs", "hbm_frac"]

MODE_BLOCK = "block-by-block"          # bench.py:24
MODE_GBG = "gate-by-gate-baseline"     # bench.py:25

SUITES = ("qubit", "scaling", "gate", "circuit", "breakdown")   # bench.py:27
GATE_FAMILIES = ("h", "rzz", "u")                               # generators.py GATE_FAMILIES
CIRCUIT_FAMILIES = ("qft", "qaoa", "bv")                        # generators.py CIRCUIT_FAMILIES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEFAULT_DIR = os.path.join(ROOT, "bench_circuits")


def _peak_gbs() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def find_circuit(family: str, n: int, r: int = 0, directory: str | None = None):
    """Path and chunk width of the optimized circuit for (family, n, r), or None."""
    d = directory or os.environ.get("QK_BENCH_CIRCUITS", DEFAULT_DIR)
    prefix = f"{family}{n}_c"
    for name in sorted(os.listdir(d)) if os.path.isdir(d) else ():
        if name.startswith(prefix) and name.endswith(f"_r{r}.txt"):
            try:
                c = int(name[len(prefix):].split("_")[0])
            except ValueError:
                continue
            return os.path.join(d, name), c
    return None


def raw_from_optimized(opt) -> RawCircuit:
    """The raw circuit behind an optimized one: gates sorted by id, targets in
    logical qubits (position -> logical map replayed through the swaps,
    circuit.py:196-210)."""
    perm = list(range(opt.num_qubits))
    gates = []
    for ins in opt.instructions:
        if isinstance(ins, GateBlock):
            for g in ins.gates:
                if g.kind is GateKind.D or g.gid is None or g.gid < 0:
                    raise ValueError("fused D<k> gates carry no id; no raw circuit")
                gates.append(Gate(g.kind, tuple(perm[t] for t in g.targets), g.gid, g.params))
        elif isinstance(ins, InMemSwap):
            apply_swap_to_permutation(perm, ins.out_set, ins.in_set)
        elif isinstance(ins, CrossRankSwap):
            apply_swap_to_permutation(perm, ins.local_set, ins.rank_set)
    gates.sort(key=lambda g: g.gid)
    return RawCircuit(opt.num_qubits, tuple(gates))


def _row(suite, workload, n, ranks, mode, reps, layout=None, **kw) -> dict:   # bench.py:43-51
    row = {"suite": suite, "workload": workload, "qubits": n, "ranks": ranks,
           "chunk_qubits": layout.c if layout else "",
           "cacheline_qubits": layout.cl if layout else "",
           "buffer_qubits": layout.b if layout else "",
           "mode": mode, "reps": reps, "mean_seconds": "", "gate_seconds": "",
           "ims_seconds": "", "xrs_seconds": "", "aio_seconds": "", "status": "ok",
           "device_seconds": "", "hbm_gbs": "", "hbm_frac": ""}
    row.update(kw)
    return row


def _time_workload(suite: str, workload: str, n: int, r: int, mode: str, reps: int,
                   directory: str | None = None) -> dict:                   # bench.py:54-86
    found = find_circuit(workload, n, r, directory)
    if found is None:
        return _row(suite, workload, n, 1 << r, mode, reps, status="missing_circuit")
    path, c = found
    text = open(path).read()
    layout = LayoutParams(n=n, c=c, r=r, b=min(n - r, 20))
    opt = parse_optimized(text, layout)
    if mode == MODE_GBG:
        if r > 0:
            return _row(suite, workload, n, 1 << r, mode, reps, layout=layout,
                        status="skipped_multirank")
        try:
            raw = raw_from_optimized(opt)
        except ValueError:
            return _row(suite, workload, n, 1, mode, reps, layout=layout, status="skipped_fused")
    totals = {"gate": 0.0, "ims": 0.0, "xrs": 0.0}
    wall = 0.0
    try:
        # one process holds every rank here; multi-GPU runs go through bench.py --gpus N
        sim = Simulator(LayoutParams(n=n, c=n - r, r=r))
    except SimulationError:
        return _row(suite, workload, n, 1 << r, mode, reps, layout=layout, status="skipped_oom")
    with sim:
        h = sim.handle
        if mode == MODE_BLOCK:
            perm = sim.load_text(text, c)
        h.stats(reset=True)
        for _ in range(reps):
            sim.reset()
            t0 = time.perf_counter()
            res = sim.run_loaded(perm) if mode == MODE_BLOCK else sim.run_gate_by_gate(raw)
            wall += time.perf_counter() - t0
            for k in totals:
                totals[k] += res.timings[k]
        st = h.stats()
    dev_ms = st[0] + st[2] + st[4] + st[9]
    alg = st[6] + st[7] + st[8] + st[11]
    gbs = alg / (dev_ms * 1e-3) / 1e9 if dev_ms else 0.0
    return _row(suite, workload, n, 1 << r, mode, reps, layout=layout,
                mean_seconds=f"{wall / reps:.6f}",
                gate_seconds=f"{totals['gate'] / reps:.6f}",
                ims_seconds=f"{totals['ims'] / reps:.6f}",
                xrs_seconds=f"{totals['xrs'] / reps:.6f}",
                aio_seconds=f"{0.0:.6f}",
                device_seconds=f"{dev_ms * 1e-3 / reps:.6f}",
                hbm_gbs=f"{gbs:.1f}", hbm_frac=f"{gbs / _peak_gbs():.4f}")


def run_bench(suite: str, *, sizes: list[int] | None = None, qubits: int = 30,
              ranks: list[int] | None = None, reps: int = 3, directory: str | None = None,
              modes: tuple = (MODE_BLOCK, MODE_GBG)) -> list[dict]:   # bench.py:89-120
    """Run one suite and return its CSV rows (reference suites, same row order)."""
    if suite not in SUITES:
        raise ValueError(f"unknown suite {suite!r}; choose from {', '.join(SUITES)}")
    rows: list[dict] = []
    if suite == "qubit":
        for n in sizes or (30, 33):
            for mode in modes:
                rows.append(_time_workload(suite, "h", n, 0, mode, reps, directory))
    elif suite == "scaling":
        for nr in ranks or (1, 2, 4, 8):
            r = nr.bit_length() - 1
            rows.append(_time_workload(suite, "qft", qubits + r, r, MODE_BLOCK, reps, directory))
    elif suite == "gate":
        for fam in GATE_FAMILIES:
            for mode in modes:
                rows.append(_time_workload(suite, fam, qubits, 0, mode, reps, directory))
    elif suite == "circuit":
        for fam in CIRCUIT_FAMILIES:
            for mode in modes:
                rows.append(_time_workload(suite, fam, qubits, 0, mode, reps, directory))
    else:  # breakdown
        for fam in CIRCUIT_FAMILIES:
            rows.append(_time_workload(suite, fam, qubits, 0, MODE_BLOCK, reps, directory))
    return rows


def rows_to_csv(rows: list[dict]) -> str:                               # bench.py:123-128
    buf = io.StringIO()
    writer = csv.DictWriter(buf, fieldnames=CSV_COLUMNS, lineterminator="\n")
    writer.writeheader()
    writer.writerows(rows)
    return buf.getvalue()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2406_14084_b200.bench")
    ap.add_argument("--suite", default="circuit", choices=SUITES)
    ap.add_argument("--qubits", type=int, default=30)
    ap.add_argument("--sizes", type=int, nargs="*")
    ap.add_argument("--ranks", type=int, nargs="*")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dir", default=None, help="directory of optimized circuits")
    ap.add_argument("--no-gbg", action="store_true", help="block-by-block rows only")
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    modes = (MODE_BLOCK,) if a.no_gbg else (MODE_BLOCK, MODE_GBG)
    rows = run_bench(a.suite, sizes=a.sizes, qubits=a.qubits, ranks=a.ranks, reps=a.reps,
                     directory=a.dir, modes=modes)
    text = rows_to_csv(rows)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
