"""CPU: host logic of the drop-in — the C ABI loads and exports every declared
symbol, the native parser follows the reference grammar and messages, the
data model validates like the reference, host bit helpers match the goldens."""
import math
import os
import re

import numpy as np
import pytest

from conftest import EXAMPLE_OPTIMIZED, ROOT
from paper_2406_14084_b200 import (CrossRankSwap, Gate, GateBlock, GateKind, InMemSwap,
                                   LayoutParams, OptimizedCircuit, ParseError, bitshift, bitswap,
                                   gate_matrix, parse_optimized, serialize_optimized)
from paper_2406_14084_b200 import _lib


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "qkb200.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(qk_\w+)\(", header, re.M))
    assert declared, "no declarations found"
    lib = _lib.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED)
    assert lib.qk_version() == 1


def test_parse_example_counts_and_permutation():
    layout = LayoutParams(n=10, c=4, r=2)
    opt = parse_optimized(EXAMPLE_OPTIMIZED, layout)
    kinds = [type(i).__name__ for i in opt.instructions]
    assert kinds.count("GateBlock") == 4 and kinds.count("InMemSwap") == 5
    assert kinds.count("CrossRankSwap") == 1
    assert opt.final_permutation == (8, 6, 9, 1, 4, 3, 5, 7, 0, 2)   # test_circuit.py:100-108


def test_parse_records():
    layout = LayoutParams(n=10, c=4, r=2)
    assert parse_optimized("1\nSQS 1 3 5", layout).instructions == (InMemSwap((3,), (5,)),)
    assert parse_optimized("1\nCSQS 2 6 7 8 9", layout).instructions == (
        CrossRankSwap((6, 7), (8, 9)),)
    (block,) = parse_optimized("2\nH 0 0\nH 1 1", layout).instructions
    assert [g.gid for g in block.gates] == [0, 1]
    assert len(parse_optimized("1 # Gate Block Size\nH 0 0 # a gate", layout).instructions) == 1
    (b2,) = parse_optimized("1\nRZZ 2 3 7", layout).instructions
    assert b2.gates[0].params == (math.pi / 4,)
    (b3,) = parse_optimized("1\nU 1 9 0.5 1.5 2.5", layout).instructions
    assert b3.gates[0].params == (0.5, 1.5, 2.5) and b3.gates[0].gid == 9


@pytest.mark.parametrize("text,message,line", [
    ("2\nH 0 0", "ends early", 1),
    ("1\nSQS 2 0 1 4", "tokens", 2),
    ("1\nH 5 0", "chunk", 2),
    ("0\nH 0 0", "positive", 1),
    ("1\nFOO 0 0", "unknown gate symbol", 2),
    ("1\nH 0 1 2 0", "token count", 2),
    ("1\nRZZ 1 1 0", "duplicate", 2),
    ("1\nH 99 0", "out of range", 2),
    ("1\nSQS 1 3 9", "outside local range", 2),
    ("1\nCSQS 1 7 2", "outside rank range", 2),
    ("H 0 0", "record count", 1),
    ("1\nH 0 -4", "negative gate id", 2),
])
def test_parse_errors(text, message, line):
    layout = LayoutParams(n=10, c=4, r=2)
    with pytest.raises(ParseError) as err:
        parse_optimized(text, layout)
    assert message in str(err.value)
    assert err.value.line_no == line


def test_round_trip_token_identical(golden):
    meta, _ = golden
    for c in meta["circuits"]:
        # no-IMS circuits hold memory-level blocks (targets >= C): parse them
        # with the whole local range as the chunk bound, like the CLI does
        layout = LayoutParams(n=c["n"], c=c["n"] - c["r"], r=c["r"], b=c["b"])
        opt = parse_optimized(c["text"], layout)
        assert serialize_optimized(opt).split() == c["text"].split(), c["name"]
        assert list(opt.final_permutation) == c["perm"]


def test_fused_gate_round_trip():
    layout = LayoutParams(n=10, c=4, r=2)
    diag = tuple(np.exp(1j * np.linspace(0, 3, 16)))
    block = GateBlock((Gate(GateKind.D, (0, 1, 2, 3), 2, diag),))
    text = serialize_optimized(OptimizedCircuit(10, layout, (block,)))
    (parsed,) = parse_optimized(text, layout).instructions
    assert np.array_equal(np.array(parsed.gates[0].params), np.array(diag))
    assert parsed.gates[0].targets == (0, 1, 2, 3)


def test_layout_and_gate_validation():
    with pytest.raises(ValueError, match="C <= N-R"):
        LayoutParams(n=4, c=5)
    with pytest.raises(ValueError, match="B <= N-R"):
        LayoutParams(n=4, c=2, r=1, b=4)
    assert LayoutParams(n=10, c=4, r=2).b == 8
    with pytest.raises(ValueError, match="duplicate"):
        Gate(GateKind.CX, (1, 1), 0)
    with pytest.raises(ValueError, match="takes 1 parameters"):
        Gate(GateKind.RZ, (1,), 0)
    with pytest.raises(ValueError, match="disjoint"):
        InMemSwap((1,), (1,))


def test_gate_matrices_match_golden(golden):
    meta, arr = golden
    for k, case in enumerate(meta["matrices"]):
        kind = GateKind(case["kind"])
        arity = 2 if case["kind"] in ("CX", "CP", "SWAP", "RZZ") else 1
        m = gate_matrix(Gate(kind, tuple(range(arity)), 0, tuple(case["params"])))
        pad = np.pad(m, ((0, 4 - m.shape[0]), (0, 4 - m.shape[1])))
        assert np.max(np.abs(pad - arr["matrices"][k])) <= 1e-16, case["kind"]


def test_bit_helpers(golden):
    meta, arr = golden
    assert bitswap(0b10000, (0,), (4,)) == 1 and bitswap(7, (), ()) == 7
    with pytest.raises(ValueError):
        bitswap(0, (0, 1), (1, 2))
    dom = np.arange(1 << 12, dtype=np.int64)
    for k, case in enumerate(meta["bitshift"]):
        out = bitshift(dom, tuple(case["a"]), tuple(case["b"]), case["cl"], 12)
        assert np.array_equal(np.asarray(out), arr["bitshift"][k])


def test_pack_round_trip():
    layout = LayoutParams(n=10, c=4, r=2)
    opt = parse_optimized(EXAMPLE_OPTIMIZED, layout)
    words, params, npar = _lib.pack(opt.instructions)
    assert words.dtype == np.int32 and npar == 6   # six RZZ angles
    assert words[0] == _lib.INS_BLOCK and words[1] == 3


def test_bench_configs_cover_baseline_and_match_between_arms():
    """bench.py: N>1 runs BASELINE C4/C5 (QFT 34/35/36 at 2/4/8 GPUs, 2^33
    amplitudes per GPU; BV/H/QAOA 36 at 8), every circuit is committed, and
    both arms print the same `config` for the same run."""
    import os
    import bench
    for fam, by_n in bench.MULTI.items():
        for world, stem in by_n.items():
            f2, n, c, r = bench.parse_stem(stem)
            assert f2 == fam and (1 << r) == world and n - r == 33, stem
            assert os.path.exists(os.path.join(bench.CIRCUITS, stem + ".txt")), stem
    assert bench.MULTI["qft"] == {2: "qft34_c10_r1", 4: "qft35_c10_r2", 8: "qft36_c10_r3"}
    for world, wl in ((1, "qaoa30"), (2, "qft"), (8, "qaoa")):
        args = type("A", (), {"circuit": None, "workload": wl})()
        name, fname, n, c, r, fam = bench.pick(args, world)
        cfg = bench.config_of(name, fname, n, c, r, world)
        assert cfg == bench.config_of(*bench.pick(args, world)[:5], world)
        assert cfg["state_bytes_per_gpu"] == 16 << (n - r)
    assert bench.analytic_factors("qaoa", 4) is None
    assert abs(np.prod(bench.analytic_factors("qft", 6)[:, 0]) - 2 ** -3) < 1e-15
