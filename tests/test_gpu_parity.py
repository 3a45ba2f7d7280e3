"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle. Permutations bit-exact; amplitudes within 1e-10
max abs (north_star tolerance; observed errors are ~1e-15)."""
import math

import numpy as np
import pytest

from conftest import EXAMPLE_OPTIMIZED, EXAMPLE_RAW  # noqa: F401
from oracle import quokka_oracle as orc
from paper_2406_14084_b200 import (CrossRankSwap, Gate, GateBlock, GateKind, InMemSwap,
                                   LayoutParams, OptimizedCircuit, SimConfig, SimulationError,
                                   Simulator, StatePartition, apply_gate_block, cross_rank_swap,
                                   get_amplitude, in_memory_swap, init_state, parse_optimized,
                                   serialize_optimized, simulate)

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _layout_for(c):
    return LayoutParams(n=c["n"], c=c["n"] - c["r"], r=c["r"], b=c["b"])


def test_golden_circuits(gpu, engine, golden):
    meta, arr = golden
    worst = 0.0
    for c in meta["circuits"]:
        layout = _layout_for(c)
        res = simulate(parse_optimized(c["text"], layout), SimConfig(layout))
        assert list(res.final_permutation) == c["perm"], c["name"]
        phys = res.physical_vector()
        if c.get("sampled"):
            err = np.max(np.abs(phys[arr[c["key"] + "_idx"]] - arr[c["key"] + "_sample"]))
        else:
            err = np.max(np.abs(phys - arr[c["key"] + "_phys"]))
        worst = max(worst, float(err))
        assert err <= TOL, (c["name"], err)
        assert abs(res.norm() - c["norm"]) <= 1e-12, c["name"]
        dense = arr.get(c["key"] + "_dense")
        if dense is not None:
            assert np.max(np.abs(res.logical_vector() - dense)) <= TOL, c["name"]
    print(f"\n  golden circuits: {len(meta['circuits'])}, worst |gpu-ref| = {worst:.3e}")


def test_golden_sqs_bit_exact(gpu, golden):
    meta, arr = golden
    for case in meta["sqs"]:
        v = np.arange(1 << case["nl"]).astype(np.complex128)
        in_memory_swap(v, tuple(case["a"]), tuple(case["b"]), case["cl"])
        want = arr["sqs_perm"][case["off"]:case["off"] + v.size]
        assert np.array_equal(v.real.astype(np.int32), want), case


def test_golden_csqs_bit_exact(gpu, golden):
    meta, arr = golden
    for case in meta["csqs"]:
        n, r = case["n"], case["r"]
        size = 1 << (n - r)
        v = np.arange(1 << n).astype(np.complex128)
        parts = [StatePartition(q, v[q * size:(q + 1) * size].copy()) for q in range(1 << r)]
        layout = LayoutParams(n=n, c=1, r=r, cl=0, b=case["b"])
        cross_rank_swap(parts, tuple(case["local"]), tuple(case["rank"]), layout)
        got = np.concatenate([p.amps for p in parts]).real.astype(np.int32)
        assert np.array_equal(got, arr["csqs_perm"][case["off"]:case["off"] + got.size]), case


def test_golden_single_blocks(gpu, golden):
    meta, arr = golden
    for case in meta["blocks"]:
        layout = LayoutParams(n=case["n"], c=case["c"])
        (block,) = parse_optimized(case["text"], layout).instructions
        part = StatePartition(0, arr[case["key"] + "_in"].copy())
        apply_gate_block(part, block, c=case["c"], cl=min(2, case["c"]))
        assert np.max(np.abs(part.amps - arr[case["key"] + "_out"])) <= TOL


# ---------------------------------------------------------------------------
# reference unit tests (pkg/tests/test_simulator.py) on the device path


def test_init_state(gpu):
    (part,) = init_state(LayoutParams(n=3, c=2))
    assert np.array_equal(part.amps, [1, 0, 0, 0, 0, 0, 0, 0])
    parts = init_state(LayoutParams(n=3, c=2, r=1))
    assert np.array_equal(parts[0].amps, [1, 0, 0, 0]) and np.array_equal(parts[1].amps, [0] * 4)
    with pytest.raises(SimulationError, match=str((1 << 40) * 16)):
        init_state(LayoutParams(n=40, c=10))


def test_block_kats(gpu):
    parts = init_state(LayoutParams(n=1, c=1, cl=0))
    apply_gate_block(parts[0], GateBlock((Gate(GateKind.H, (0,), 0),)), c=1, cl=0)
    assert np.allclose(np.asarray(parts[0].amps), [2 ** -0.5, 2 ** -0.5])
    part = StatePartition(0, np.zeros(4, dtype=complex))
    part.amps[0b01] = 1.0
    apply_gate_block(part, GateBlock((Gate(GateKind.CX, (0, 1), 0),)), c=2, cl=0)
    assert part.amps[0b11] == 1.0 and part.amps[0b01] == 0.0
    rng = np.random.default_rng(1)
    v = rng.normal(size=16) + 1j * rng.normal(size=16)
    part = StatePartition(0, v.copy())
    apply_gate_block(part, GateBlock((Gate(GateKind.H, (0,), 0), Gate(GateKind.H, (0,), 1))),
                     c=2, cl=0)
    assert np.max(np.abs(part.amps - v)) <= 1e-15
    with pytest.raises(SimulationError):
        apply_gate_block(StatePartition(0, np.zeros(8, dtype=complex)),
                         GateBlock((Gate(GateKind.H, (2,), 0),)), c=2, cl=0)


def test_sqs_kats_and_ranges(gpu):
    amps = np.array([1, 2, 3, 4], dtype=complex)
    in_memory_swap(amps, (0,), (1,), cl=0)
    assert np.array_equal(amps, [1, 3, 2, 4])
    rng = np.random.default_rng(9)
    v = rng.normal(size=1 << 10) + 1j * rng.normal(size=1 << 10)
    whole = v.copy()
    in_memory_swap(whole, (1, 4), (6, 8), cl=2)
    assert np.array_equal(whole, orc.bitswap_permute(v, (1, 4), (6, 8)))
    pieces = v.copy()
    cut = int(rng.integers(1, 1 << 10))
    in_memory_swap(pieces, (1, 4), (6, 8), cl=2, start=0, stop=cut)
    in_memory_swap(pieces, (1, 4), (6, 8), cl=2, start=cut)
    assert np.array_equal(whole, pieces)
    with pytest.raises(ValueError, match="out of range"):
        in_memory_swap(np.zeros(8, dtype=complex), (0,), (3,), cl=0)


def test_csqs_contract_checks(gpu):
    layout = LayoutParams(n=6, c=2, r=2, b=1)
    parts = init_state(layout)
    with pytest.raises(SimulationError, match="top-of-local"):
        cross_rank_swap(parts, (0, 1), (4, 5), layout)
    with pytest.raises(SimulationError, match="buffer"):
        cross_rank_swap(parts, (2, 3), (4, 5), layout)


def test_executor_semantics(gpu):
    layout = LayoutParams(n=4, c=2)
    with Simulator(layout) as sim:
        res = sim.run([])
        assert np.array_equal(res.partitions[0].amps[:2], [1, 0])
        assert res.norm() == 1.0
    layout = LayoutParams(n=2, c=1, cl=0)
    parts = init_state(layout)
    parts[0].amps[:] = [0, 0.5, 0.25, 0]
    assert get_amplitude(parts, 0b01, (1, 0)) == 0.25
    assert get_amplitude(parts, 0b10, (1, 0)) == 0.5
    # memory-level path for a wide block (test_simulator.py:376-386)
    layout = LayoutParams(n=6, c=2)
    rng = np.random.default_rng(16)
    v = rng.normal(size=64) + 1j * rng.normal(size=64)
    with Simulator(layout) as sim:
        sim.partitions[0].amps[:] = v
        res = sim.run([GateBlock((Gate(GateKind.H, (5,), 0),))])
    want = v.copy().reshape(2, 32)
    want = np.vstack([(want[0] + want[1]), (want[0] - want[1])]) * 2 ** -0.5
    assert np.max(np.abs(np.asarray(res.partitions[0].amps) - want.reshape(-1))) <= 1e-15
    with pytest.raises(SimulationError, match="qubits"):
        Simulator(LayoutParams(n=5, c=2)).run(OptimizedCircuit(4, LayoutParams(n=4, c=2), ()))


def test_gate_by_gate_matches_block_mode(gpu):
    text = "\n".join(f"H {q} {q}" for q in range(9))
    from paper_2406_14084_b200 import RawCircuit
    raw = RawCircuit(9, tuple(Gate(GateKind.H, (q,), q) for q in range(9)) +
                     (Gate(GateKind.CP, (0, 8), 9, (0.3,)), Gate(GateKind.RX, (8,), 10, (1.1,))))
    with Simulator(LayoutParams(n=9, c=4)) as sim:
        res = sim.run_gate_by_gate(raw)
        got = res.logical_vector()
    state = np.zeros(512, complex)
    state[0] = 1
    for g in raw.gates:
        state = orc.dense_apply(state, orc.OGate(g.kind.value, g.targets, g.gid, g.params), 9)
    assert np.max(np.abs(got - state)) <= TOL
    assert text  # keeps the H-layer recipe visible
    with pytest.raises(SimulationError):
        Simulator(LayoutParams(n=6, c=2, r=1)).run_gate_by_gate(raw)


# ---------------------------------------------------------------------------
# randomized instruction streams vs the oracle (all gate kinds, D<k>, SQS, CSQS,
# memory-level blocks, chunk widths up to 13)

KINDS = ["H", "X", "U", "CX", "CP", "SWAP", "RX", "RY", "RZ", "RZZ", "D"]


def _random_gate(rng, c, gid):
    kind = KINDS[rng.integers(0, len(KINDS))]
    if kind == "D" and c < 2:
        kind = "RZ"
    if kind == "D":
        k = int(rng.integers(2, min(c, 6) + 1))
        t = tuple(int(x) for x in np.sort(rng.choice(c, size=k, replace=False)))
        return Gate(GateKind.D, t, gid, tuple(np.exp(1j * rng.uniform(0, 2 * np.pi, 1 << k))))
    arity = 2 if kind in ("CX", "CP", "SWAP", "RZZ") else 1
    if arity > c:
        kind, arity = "H", 1
    t = tuple(int(x) for x in rng.choice(c, size=arity, replace=False))
    npar = {"U": 3, "CP": 1, "RX": 1, "RY": 1, "RZ": 1, "RZZ": 1}.get(kind, 0)
    return Gate(GateKind(kind), t, gid, tuple(float(a) for a in rng.uniform(0, 2 * np.pi, npar)))


def _random_stream(rng, n, r, c, nins, mem_level=True):
    L = n - r
    out, gid = [], 0
    for _ in range(nins):
        roll = rng.random()
        if roll < 0.55 or L < 2:
            width = c if (rng.random() < 0.85 or not mem_level) else L  # some memory-level blocks
            gates = []
            for _ in range(int(rng.integers(1, 40))):
                gates.append(_random_gate(rng, width, gid))
                gid += 1
            out.append(GateBlock(tuple(gates)))
        elif roll < 0.85 or r == 0:
            k = int(rng.integers(1, L // 2 + 1))
            bits = rng.choice(L, size=2 * k, replace=False)
            out.append(InMemSwap(tuple(int(x) for x in bits[:k]), tuple(int(x) for x in bits[k:])))
        else:
            s = int(rng.integers(1, min(r, L) + 1))
            rank = tuple(int(x) for x in np.sort(rng.choice(np.arange(L, n), size=s, replace=False)))
            out.append(CrossRankSwap(tuple(range(L - s, L)), rank))
    return tuple(out)


@pytest.fixture(params=["interp", "jit"])
def engine(request):
    """Run a test once with the interpreted passes and once with every TMA pass
    specialised by the load-time JIT (QK_JIT=<min address bits>)."""
    import os
    if request.param == "jit":
        os.environ["QK_JIT"] = "0"
    else:
        os.environ["QK_JIT"] = "99"
    yield request.param
    os.environ.pop("QK_JIT", None)


@pytest.mark.parametrize("seed", range(24))
def test_random_streams_vs_oracle(gpu, engine, seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(3, 15))
    r = int(rng.integers(0, min(3, n - 1) + 1))
    L = n - r
    c = int(rng.integers(1, min(L, 13) + 1))
    b = int(rng.integers(min(r, L), L + 1)) if r else L
    layout = LayoutParams(n=n, c=L, r=r, cl=min(2, L), b=b)
    ins = _random_stream(rng, n, r, c, int(rng.integers(1, 16)))
    opt = OptimizedCircuit(n, layout, ins)
    text = serialize_optimized(opt)
    if not ins:
        return
    # CSQS with B < S is a contract error in both
    need_b = max((len(i.local_set) for i in ins if isinstance(i, CrossRankSwap)), default=0)
    if need_b > b:
        with pytest.raises(SimulationError):
            simulate(opt, SimConfig(layout))
        return
    res = simulate(opt, SimConfig(layout))
    want, perm, _ = orc.simulate_text(text, n, L, r=r, b=b)
    assert tuple(res.final_permutation) == perm
    err = float(np.max(np.abs(res.physical_vector() - want)))
    assert err <= TOL, (seed, n, r, c, err)


@pytest.mark.parametrize("seed", range(10))
def test_random_streams_in_the_scheduled_range_vs_oracle(gpu, seed):
    """Random instruction streams at 17-21 qubits with chunks of 8-12 (QK_JIT=0:
    the lazy layout and the cross-block schedule apply from 16 address bits),
    half of them without D<k> gates so the schedule, the quadratic phases, the
    zero-support reads and chunk skipping and the first-use placement all run
    (every block chunked except in one seed of four); R = 0..2 rank partitions
    in one handle. Against the oracle; the plan summary must show the schedule
    (QK_DUMP_PLAN) for the seeds that allow it."""
    import os
    rng = np.random.default_rng(9100 + seed)
    n = int(rng.integers(17, 22))
    r = int(rng.integers(0, 3))
    L = n - r
    c = int(rng.integers(8, 13))
    layout = LayoutParams(n=n, c=L, r=r, cl=2, b=L)
    global KINDS
    kinds0 = KINDS
    if seed % 2 == 0:
        KINDS = [k for k in KINDS if k != "D"]
    try:
        ins = _random_stream(rng, n, r, c, int(rng.integers(4, 14)), mem_level=seed % 4 == 3)
    finally:
        KINDS = kinds0
    text = serialize_optimized(OptimizedCircuit(n, layout, ins))
    os.environ["QK_JIT"] = "0"
    try:
        res = simulate(OptimizedCircuit(n, layout, ins), SimConfig(layout))
        got = res.physical_vector()
    finally:
        os.environ.pop("QK_JIT", None)
    want, perm, _ = orc.simulate_text(text, n, L, r=r, b=L)
    assert tuple(res.final_permutation) == perm
    err = float(np.max(np.abs(got - want)))
    assert err <= TOL, (seed, n, r, c, err)


def test_chunk_widths_up_to_13(gpu, engine):
    rng = np.random.default_rng(77)
    for c in (10, 11, 12, 13):
        n = 16
        gates = tuple(_random_gate(rng, c, i) for i in range(60))
        layout = LayoutParams(n=n, c=c)
        opt = OptimizedCircuit(n, layout, (GateBlock(gates),))
        res = simulate(opt, SimConfig(layout))
        want, _, _ = orc.simulate_text(serialize_optimized(opt), n, c)
        assert np.max(np.abs(res.physical_vector() - want)) <= TOL, c


# ---------------------------------------------------------------------------
# size-independent properties at larger sizes


def test_h_layer_uniform_and_involutions_at_28_qubits(gpu):
    n = 28
    layout = LayoutParams(n=n, c=10)
    # H on every qubit via blocks of 10 + SQS, written directly
    ins = []
    for lo in range(0, n, 10):
        qs = list(range(lo, min(lo + 10, n)))
        if lo:
            ins.append(InMemSwap(tuple(range(len(qs))), tuple(qs)))
        ins.append(GateBlock(tuple(Gate(GateKind.H, (q,), q) for q in range(len(qs)))))
    with Simulator(layout) as sim:
        res = sim.run(ins)
        amp = 2 ** (-n / 2)
        sample = res.partitions[0].amps[:4096]
        assert np.max(np.abs(sample - amp)) <= 1e-15
        assert abs(res.norm() - 1.0) <= 1e-12
        # SQS twice is the identity, bit-exact, on a random state prefix check
        rng = np.random.default_rng(3)
        head = rng.normal(size=1 << 16) + 1j * rng.normal(size=1 << 16)
        sim.partitions[0].amps[:1 << 16] = head
        sim.run([InMemSwap((0, 3, 17), (27, 9, 20))] * 2)
        assert np.array_equal(sim.partitions[0].amps[:1 << 16], head)
        sim.partitions[0].amps[:1 << 16] = head
        sim.run([InMemSwap((0, 3, 17), (27, 9, 20))])
        idx = np.arange(1 << 16)
        src = orc.bitswap(idx, (0, 3, 17), (27, 9, 20))
        inside = src < (1 << 16)
        got = sim.partitions[0].amps[idx[inside]]
        assert np.array_equal(got, head[src[inside]])


def test_bv_basis_state_30_qubits(gpu):
    import os
    from conftest import ROOT
    text = open(os.path.join(ROOT, "bench_circuits", "bv30_c10_r0.txt")).read()
    layout = LayoutParams(n=30, c=30)
    res = simulate(parse_optimized(text, layout), SimConfig(layout))
    # BV (all-ones secret, target in |+>): the state returns to the basis
    # state |0...0> (reference test_oracle.py:37-42)
    amps = res.logical_amplitudes(8)
    assert abs(res.norm() - 1.0) <= 1e-12
    assert abs(abs(amps[0]) - 1.0) <= 1e-12 and np.max(np.abs(amps[1:])) <= 1e-12
    assert abs(res.amplitude((1 << 30) - 1)) <= 1e-12
    assert math.isfinite(res.timings["gate"])


# ---------------------------------------------------------------------------
# at scale: every execution strategy must agree (persistent-ring stage reuse,
# fused out-of-place SQS, cluster-exchange SQS, interpreter fallback) on
# reference-optimized circuits


@pytest.mark.parametrize("name,n,c", [("qaoa24_c12_r0", 24, 12), ("qaoa26_c12_r0", 26, 12),
                                      ("qft26_c10_r0", 26, 10)])
def test_execution_strategies_agree_at_scale(gpu, name, n, c):
    import os
    from conftest import ROOT
    text = open(os.path.join(ROOT, "bench_circuits", name + ".txt")).read()
    outs = {}
    modes = ("default", "QK_XFUSE_ALL", "QK_NO_XFUSE", "QK_NO_FUSE", "QK_NO_TMA", "QK_NO_JIT",
             "QK_INPLACE+QK_JIT=0", "QK_INPLACE+QK_JIT=0+QK_NO_LAZY_PERM", "QK_INPLACE+QK_NO_LAZY")
    for mode in modes:
        envs = [] if mode == "default" else [e.partition("=") for e in mode.split("+")]
        for k, _, v in envs:
            os.environ[k] = v or "1"
        try:
            sim = Simulator(LayoutParams(n=n, c=n))
            perm = sim.load_text(text, c)
            for _ in range(2):            # second run reuses every ring stage again
                sim.handle.reset()
                res = sim.run_loaded(perm)
            outs[mode] = res.physical_vector()
            assert abs(res.norm() - 1.0) <= 1e-12, (mode, res.norm())
        finally:
            for k, _, _ in envs:
                os.environ.pop(k, None)
    base = outs["QK_NO_TMA"]
    for mode, vec in outs.items():
        assert np.max(np.abs(vec - base)) <= TOL, mode


@pytest.mark.gpu
def test_lazy_layout_readbacks_and_writers(gpu):
    """In-place states keep SQS as a layout relabeling (no second buffer; forced
    here at 24 qubits): every readback maps through the layout, a second run
    and kernel-level writers first restore the reference layout. All of it
    must match a handle that executes every swap."""
    import os
    from conftest import ROOT
    text = open(os.path.join(ROOT, "bench_circuits", "qaoa24_c12_r0.txt")).read()
    n = 24
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 1 << n, size=64)

    def session(env):
        for k, v in env.items():
            os.environ[k] = v
        try:
            sim = Simulator(LayoutParams(n=n, c=n))
            perm = sim.load_text(text, 12)
            sim.handle.reset()
            res = sim.run_loaded(perm)
            out = {"phys": res.physical_vector(), "norm": res.norm(),
                   "amp": [res.amplitude(int(i)) for i in idx[:8]],
                   "logical": res.logical_amplitudes(4096, start=12345),
                   "slice": np.array(res.partitions[0].amps[1000:1064])}
            res2 = sim.run_loaded(perm)          # no reset: continues from the end layout
            out["twice"] = res2.physical_vector()
            in_memory_swap(sim.partitions[0].amps, (0, 5), (7, 20), 2)   # kernel-level writer
            out["after_sqs"] = sim.partitions[0].amps[:]
            sim.close()
            return out
        finally:
            for k in env:
                os.environ.pop(k, None)

    lazy = session({"QK_INPLACE": "1", "QK_JIT": "0"})
    eager = session({"QK_NO_TMA": "1"})
    for key in ("phys", "logical", "slice", "twice", "after_sqs"):
        assert np.max(np.abs(np.asarray(lazy[key]) - np.asarray(eager[key]))) <= TOL, key
    assert abs(lazy["norm"] - eager["norm"]) <= 1e-12
    assert np.max(np.abs(np.array(lazy["amp"]) - np.array(eager["amp"]))) <= TOL


@pytest.mark.gpu
def test_fresh_reset_readers_writers_and_first_pass(gpu):
    """qk_reset writes only the first chunk of |0...0>: the first TMA pass reads
    every other chunk as out-of-bounds zeros, and any other reader or writer
    fills the whole state first. Every path must equal a handle that always
    writes the whole state (QK_NO_FRESH)."""
    import os
    from conftest import ROOT
    from paper_2406_14084_b200 import InMemSwap
    n = 20
    text = open(os.path.join(ROOT, "bench_circuits", "qft20_c10_r0.txt")).read()
    e0 = np.zeros(1 << n, dtype=np.complex128)
    e0[0] = 1

    def session(env):
        for k, v in env.items():
            os.environ[k] = v
        try:
            out = {}
            sim = Simulator(LayoutParams(n=n, c=n))
            sim.reset()
            out["read_after_reset"] = sim.partitions[0].amps[:]
            sim.reset()
            out["norm_after_reset"] = sim.handle.sumsq()
            sim.reset()
            sim.partitions[0].amps[3:7] = np.arange(4) + 1j         # partial writer
            out["after_write"] = sim.partitions[0].amps[:]
            perm = sim.load_text(text, 10)
            sim.reset()
            out["run"] = sim.run_loaded(perm).physical_vector()
            # a program that starts with a swap, then gates
            prog = [InMemSwap((0, 1), (15, 19)),
                    GateBlock(tuple(Gate(GateKind.H, (q,), q) for q in range(10)))]
            sim.reset()
            out["swap_first"] = sim.run(prog).physical_vector()
            sim.close()
            return out
        finally:
            for k in env:
                os.environ.pop(k, None)

    # (variants pinned: the comparison is bit for bit)
    fresh = session({"QK_NO_TUNE": "1"})
    full = session({"QK_NO_FRESH": "1", "QK_NO_TUNE": "1"})
    assert np.array_equal(fresh["read_after_reset"], e0)
    assert abs(fresh["norm_after_reset"] - 1.0) <= 1e-15
    want = e0.copy()
    want[3:7] = np.arange(4) + 1j
    assert np.array_equal(fresh["after_write"], want)
    for key in ("read_after_reset", "after_write", "run", "swap_first"):
        assert np.array_equal(np.asarray(fresh[key]), np.asarray(full[key])), key


@pytest.mark.gpu
def test_wide_chunk_lazy_layout_at_33_qubits(gpu):
    """QAOA33 c12 with 8 rank partitions in one 128-GiB handle: the lazy layout
    with fix-up swaps, the table-aware chunk order and the shared-memory table
    slices (states of >= 2^32 amplitudes only) against the eager mode that
    executes every swap (sampled physical amplitudes and the norm)."""
    import gc
    import os
    from conftest import ROOT
    text = open(os.path.join(ROOT, "bench_circuits", "qaoa33_c12_r3.txt")).read()
    n, r = 33, 3
    idx = np.random.default_rng(11).integers(0, 1 << n, size=1 << 16, dtype=np.uint64)

    def session(env):
        for k, v in env.items():
            os.environ[k] = v
        try:
            sim = Simulator(LayoutParams(n=n, c=n - r, r=r))
            perm = sim.load_text(text, 12)
            sim.reset()
            res = sim.run_loaded(perm)
            out = (sim.handle.gather(idx), res.norm())
            sim.close()
            del res, sim
            gc.collect()
            return out
        finally:
            for k in env:
                os.environ.pop(k, None)

    lazy = session({})
    eager = session({"QK_NO_LAZY12": "1"})
    assert np.max(np.abs(lazy[0] - eager[0])) <= TOL
    assert abs(lazy[1] - eager[1]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["default", "eager", "block_order", "no_zbound"])
def test_fused_norm_matches_full_sum_and_invalidates(gpu, mode):
    """The run's last pass sums |amp|^2 of what it stores; qk_sumsq then only
    adds the per-group partials. It must equal the full-state sum, and any
    later writer must fall back to the full sum. Every store path: the lazy
    layout with the cross-block schedule (default), the relabeled/eager modes
    (QK_NO_LAZY12), the optimizer's block order (QK_NO_REBLOCK), full reads
    after the first pass (QK_NO_ZBOUND), and a 2^30-amplitude state."""
    import os
    from conftest import ROOT
    env = {"eager": {"QK_NO_LAZY12": "1"}, "block_order": {"QK_NO_REBLOCK": "1"},
           "no_zbound": {"QK_NO_ZBOUND": "1"}}.get(mode, {})
    cases = [("qaoa24_c12_r0.txt", 24, 12), ("qft20_c10_r0.txt", 20, 10)]
    if mode in ("default", "eager"):
        cases.append(("qaoa30_c12_r0.txt", 30, 12))
    os.environ.update(env)
    try:
        _fused_norm_cases(cases, ROOT)
    finally:
        for k in env:
            os.environ.pop(k, None)


def _fused_norm_cases(cases, ROOT):
    import os
    for name, n, c in cases:
        text = open(os.path.join(ROOT, "bench_circuits", name)).read()
        sim = Simulator(LayoutParams(n=n, c=n))
        perm = sim.load_text(text, c)
        sim.reset()
        sim.run_loaded(perm)
        fused = sim.handle.sumsq()
        os.environ["QK_NO_FUSED_NORM"] = "1"
        try:
            full = sim.handle.sumsq()
        finally:
            os.environ.pop("QK_NO_FUSED_NORM")
        assert abs(fused - full) <= 1e-12, (name, fused, full)
        sim.partitions[0].amps[0:1] = np.array([3.0 + 4.0j])   # a writer: |a0|^2 becomes 25
        after = sim.handle.sumsq()
        os.environ["QK_NO_FUSED_NORM"] = "1"
        try:
            want = sim.handle.sumsq()
        finally:
            os.environ.pop("QK_NO_FUSED_NORM")
        assert after == want and after > 20.0
        sim.release()
