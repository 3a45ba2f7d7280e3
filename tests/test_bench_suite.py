"""Benchmark suites with the reference's CSV schema (paper_2406_14084_b200.bench,
mirroring /root/reference/pkg/src/quokka/bench.py)."""
import csv
import io

import numpy as np
import pytest

from conftest import EXAMPLE_OPTIMIZED, EXAMPLE_RAW
from paper_2406_14084_b200 import LayoutParams, Simulator, parse_optimized
from paper_2406_14084_b200 import bench as qb

# reference bench.py:19-22
REFERENCE_COLUMNS = ["suite", "workload", "qubits", "ranks", "chunk_qubits",
                     "cacheline_qubits", "buffer_qubits", "mode", "reps",
                     "mean_seconds", "gate_seconds", "ims_seconds", "xrs_seconds",
                     "aio_seconds", "status"]

SYMMETRIC = {"RZZ", "CP", "SWAP"}


def test_csv_schema_extends_reference():
    assert qb.CSV_COLUMNS[:len(REFERENCE_COLUMNS)] == REFERENCE_COLUMNS
    assert qb.MODE_BLOCK == "block-by-block" and qb.MODE_GBG == "gate-by-gate-baseline"
    assert qb.SUITES == ("qubit", "scaling", "gate", "circuit", "breakdown")
    text = qb.rows_to_csv([qb._row("circuit", "qft", 20, 1, qb.MODE_BLOCK, 3,
                                   status="missing_circuit")])
    rows = list(csv.DictReader(io.StringIO(text)))
    assert rows[0]["status"] == "missing_circuit" and rows[0]["mode"] == "block-by-block"


def test_unknown_suite_rejected():
    with pytest.raises(ValueError, match="unknown suite"):
        qb.run_bench("nope")


def test_raw_circuit_rebuilt_from_optimized_example():
    """reference conftest example: raw gates (ids, logical targets) come back
    from the optimized text through the swap replay."""
    opt = parse_optimized(EXAMPLE_OPTIMIZED, LayoutParams(n=10, c=4, r=2, b=8))
    raw = qb.raw_from_optimized(opt)
    want = []
    for line in EXAMPLE_RAW.strip().splitlines():
        f = line.split()
        want.append((f[0], tuple(int(x) for x in f[1:-1]), int(f[-1])))
    got = [(g.kind.value, g.targets, g.gid) for g in raw.gates]
    assert len(got) == len(want)
    for (gk, gt, gi), (wk, wt, wi) in zip(got, want):
        assert (gk, gi) == (wk, wi)
        assert (sorted(gt) if gk in SYMMETRIC else gt) == (sorted(wt) if wk in SYMMETRIC else wt)


def test_find_committed_circuits():
    path, c = qb.find_circuit("qaoa", 30)
    assert path.endswith("qaoa30_c12_r0.txt") and c == 12
    assert qb.find_circuit("qft", 34, 1)[1] == 10
    assert qb.find_circuit("qft", 99) is None


@pytest.mark.gpu
def test_gate_by_gate_baseline_matches_block_mode(gpu):
    """GBG on the rebuilt raw circuit (logical layout) equals the block-mode
    state read back in logical order (simulator.py:557-569)."""
    path, c = qb.find_circuit("qft", 20)
    text = open(path).read()
    opt = parse_optimized(text, LayoutParams(n=20, c=c))
    sim = Simulator(LayoutParams(n=20, c=c))
    block = sim.run(opt).logical_vector()
    sim.reset()
    raw = qb.raw_from_optimized(opt)
    sim.handle.stats(reset=True)
    gbg = sim.run_gate_by_gate(raw).physical_vector()
    assert np.max(np.abs(block - gbg)) <= 1e-10
    # the baseline sweeps the state once per gate: nothing fused or folded
    assert sim.handle.stats()[1] == len(raw.gates)
    sim.close()


@pytest.mark.gpu
def test_circuit_suite_rows(gpu):
    rows = qb.run_bench("circuit", qubits=20, reps=2)
    by = {(r["workload"], r["mode"]): r for r in rows}
    assert [r["workload"] for r in rows] == ["qft", "qft", "qaoa", "qaoa", "bv", "bv"]
    for mode in (qb.MODE_BLOCK, qb.MODE_GBG):
        r = by[("qft", mode)]
        assert r["status"] == "ok", r
        assert float(r["mean_seconds"]) > 0 and float(r["hbm_gbs"]) > 0
        assert r["chunk_qubits"] == 10 and r["aio_seconds"] == "0.000000"
    assert by[("qaoa", qb.MODE_BLOCK)]["status"] == "missing_circuit"
