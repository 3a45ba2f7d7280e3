"""CUDA-graph replay of small runs (qk_run → graph_run in csrc/qk_runtime.cpp):
the launches of a run from one start state are captured once and replayed.
A replayed run must equal an eager run (QK_NO_GRAPH) bit for bit from every
start state: after reset (zero-support views), from a written state, and
chained runs without a reset in between; and the result must match the
oracle / analytic answer like any run (simulator.py:529-555)."""
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import quokka_oracle as orc
from paper_2406_14084_b200 import LayoutParams, Simulator

pytestmark = pytest.mark.gpu


def _session(text, n, c, env, seed=7):
    for k, v in env.items():
        os.environ[k] = v
    try:
        out = {}
        sim = Simulator(LayoutParams(n=n, c=n))
        perm = sim.load_text(text, c)
        sim.handle.stats(reset=True)
        for k in range(4):                               # after reset: capture, then replays
            sim.reset()
            res = sim.run_loaded(perm)
            out[f"reset{k}"] = res.physical_vector()
            assert sum(res.timings.values()) > 0
        rng = np.random.default_rng(seed)
        v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        v /= np.linalg.norm(v)
        out["input"] = v
        for k in range(3):                               # from a written state
            sim.partitions[0].amps[:] = v
            out[f"written{k}"] = sim.run_loaded(perm).physical_vector()
        sim.reset()
        for k in range(3):                               # chained runs, no reset
            out[f"chain{k}"] = sim.run_loaded(perm).physical_vector()
        out["replays"] = sim.handle.stats()[13]
        out["norm"] = sim.handle.sumsq()
        sim.close()
        return out
    finally:
        for k in env:
            os.environ.pop(k, None)


@pytest.mark.parametrize("name,n,c", [("qft20_c10_r0", 20, 10), ("qaoa24_c12_r0", 24, 12)])
def test_graph_replay_equals_eager(gpu, name, n, c):
    text = open(os.path.join(ROOT, "bench_circuits", name + ".txt")).read()
    g = _session(text, n, c, {"QK_NO_TUNE": "1"})
    e = _session(text, n, c, {"QK_NO_TUNE": "1", "QK_NO_GRAPH": "1"})
    # 4 runs after reset, 3 from a written state: the first of each start state
    # runs eagerly, the second captures (chained runs replay when the run ends
    # in the reference layout)
    assert g["replays"] >= 5, g["replays"]
    assert e["replays"] == 0
    for key in g:
        if key.startswith(("reset", "written", "chain")):
            assert np.array_equal(g[key], e[key]), key
    for k in range(1, 4):
        assert np.array_equal(g["reset0"], g[f"reset{k}"])
    for k in range(1, 3):
        assert np.array_equal(g["written0"], g[f"written{k}"])
    assert abs(g["norm"] - 1.0) <= 1e-10
    if n <= 20:  # the oracle from the same written state and from |0...0>
        instrs = orc.parse_optimized_text(text, n, c, n)
        osim = orc.OracleSimulator(n, c)
        osim.parts[0][:] = g["input"]
        osim.run(instrs)
        assert np.max(np.abs(g["written0"] - osim.physical())) <= 1e-10
        want, _, _ = orc.simulate_text(text, n, c)
        assert np.max(np.abs(g["reset3"] - want)) <= 1e-10


def test_graph_after_tuning_and_not_for_large_states(gpu):
    """Autotuning runs stay eager (their variants are timed per pass; the tune
    record is process-wide, so an earlier test may have finished it), later
    runs replay; a state above 2^QK_GRAPH_BITS (24) is never captured."""
    text = open(os.path.join(ROOT, "bench_circuits", "qft20_c10_r0.txt")).read()
    sim = Simulator(LayoutParams(n=20, c=20))
    perm = sim.load_text(text, 10)
    sim.handle.stats(reset=True)
    for _ in range(40):
        sim.reset()
        last = sim.run_loaded(perm).physical_vector()
    assert sim.handle.stats()[13] > 0
    assert np.max(np.abs(np.abs(last) - 2.0 ** -10)) <= 1e-12  # QFT of |0...0>: uniform magnitudes
    # a load per run (the e2e path), alternating with another program: the
    # same plan uploaded again keeps its graph, the other one gets its own
    from paper_2406_14084_b200 import Gate, GateBlock, GateKind, InMemSwap
    other = [InMemSwap((0, 1), (15, 19)),
             GateBlock(tuple(Gate(GateKind.H, (q,), q) for q in range(10)))]
    sim.reset()
    want_other = sim.run(other).physical_vector()
    sim.handle.stats(reset=True)
    for _ in range(4):
        perm = sim.load_text(text, 10)
        sim.reset()
        assert np.array_equal(sim.run_loaded(perm).physical_vector(), last)
        sim.reset()
        assert np.array_equal(sim.run(other).physical_vector(), want_other)
    assert sim.handle.stats()[13] > 0
    sim.close()
    text = open(os.path.join(ROOT, "bench_circuits", "qft26_c10_r0.txt")).read()
    os.environ["QK_NO_TUNE"] = "1"
    try:
        sim = Simulator(LayoutParams(n=26, c=26))
        perm = sim.load_text(text, 10)
        sim.handle.stats(reset=True)
        for _ in range(3):
            sim.reset()
            sim.run_loaded(perm)
        assert sim.handle.stats()[13] == 0
        assert abs(sim.handle.sumsq() - 1.0) <= 1e-10
        sim.close()
    finally:
        os.environ.pop("QK_NO_TUNE", None)
