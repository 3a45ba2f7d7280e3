"""CPU: the numpy oracle (oracle/quokka_oracle.py) pinned against vectors the
reference itself produced (oracle/gen_golden.py). No GPU needed."""
import numpy as np
import pytest

from oracle import quokka_oracle as orc


def _run_case(c):
    return orc.simulate_text(c["text"], c["n"], c["c"], r=c["r"], b=c["b"], cl=c["cl"])


def test_oracle_reproduces_every_golden_circuit(golden):
    meta, arr = golden
    worst = 0.0
    for c in meta["circuits"]:
        phys, perm, _ = _run_case(c)
        assert list(perm) == c["perm"], c["name"]
        if c.get("sampled"):
            got = phys[arr[c["key"] + "_idx"]]
            want = arr[c["key"] + "_sample"]
        else:
            got, want = phys, arr[c["key"] + "_phys"]
        err = float(np.max(np.abs(got - want)))
        worst = max(worst, err)
        assert err <= 1e-12, (c["name"], err)
        assert abs(orc.norm([phys]) - c["norm"]) <= 1e-12
    assert worst <= 1e-12


def test_oracle_matches_dense_reference(golden):
    meta, arr = golden
    for c in meta["circuits"]:
        key = c["key"] + "_dense"
        if key not in arr:
            continue
        phys, perm, _ = _run_case(c)
        logical = orc.logical_state(phys, perm)
        assert np.max(np.abs(logical - arr[key])) <= 1e-12, c["name"]


def test_oracle_sqs_permutations_bit_exact(golden):
    meta, arr = golden
    perms = arr["sqs_perm"]
    for case in meta["sqs"]:
        v = np.arange(1 << case["nl"]).astype(np.complex128)
        orc.in_memory_swap(v, tuple(case["a"]), tuple(case["b"]), case["cl"])
        want = perms[case["off"]:case["off"] + v.size]
        assert np.array_equal(v.real.astype(np.int32), want)


def test_oracle_csqs_permutations_bit_exact(golden):
    meta, arr = golden
    perms = arr["csqs_perm"]
    for case in meta["csqs"]:
        n, r = case["n"], case["r"]
        size = 1 << (n - r)
        v = np.arange(1 << n).astype(np.complex128)
        parts = [v[q * size:(q + 1) * size].copy() for q in range(1 << r)]
        orc.cross_rank_swap(parts, tuple(case["local"]), tuple(case["rank"]), n, r, case["b"])
        got = np.concatenate(parts).real.astype(np.int32)
        assert np.array_equal(got, perms[case["off"]:case["off"] + got.size])


def test_oracle_bitshift_and_matrices(golden):
    meta, arr = golden
    dom = np.arange(1 << 12, dtype=np.int64)
    for k, case in enumerate(meta["bitshift"]):
        out = orc.bitshift(dom, tuple(case["a"]), tuple(case["b"]), case["cl"], 12)
        assert np.array_equal(np.asarray(out), arr["bitshift"][k])
    for k, case in enumerate(meta["matrices"]):
        m = orc.gate_matrix(case["kind"], case["params"])
        pad = np.pad(m, ((0, 4 - m.shape[0]), (0, 4 - m.shape[1])))
        assert np.array_equal(pad, arr["matrices"][k]), case["kind"]


def test_oracle_single_blocks(golden):
    meta, arr = golden
    for case in meta["blocks"]:
        instrs = orc.parse_optimized_text(case["text"], case["n"], case["c"], case["n"])
        v = arr[case["key"] + "_in"].copy()
        orc.apply_block_rows(v, instrs[0][1], case["c"])
        assert np.max(np.abs(v - arr[case["key"] + "_out"])) <= 1e-15


def test_oracle_analytic_answers():
    # QFT|0> is uniform; H layer is uniform (test_oracle.py:32-42 analogues)
    from paper_2406_14084_b200 import LayoutParams  # noqa: F401  (layout semantics only)
    n = 6
    text = "\n".join(["%d" % n] + [f"H {q} {q}" for q in range(n)])
    phys, _, _ = orc.simulate_text(text, n, n)
    assert np.allclose(phys, 2 ** (-n / 2), atol=1e-15)


def test_oracle_contract_errors():
    with pytest.raises(orc.OracleError, match="top-of-local"):
        parts = [np.zeros(16, complex) for _ in range(4)]
        orc.cross_rank_swap(parts, (0, 1), (4, 5), 6, 2, 1)
    with pytest.raises(ValueError, match="out of range"):
        orc.in_memory_swap(np.zeros(8, complex), (0,), (3,))
