"""GPU, two processes sharing cuda:0: the multi-process shard path end to end.

Each process owns half of the 2^R rank partitions (qk_create_shard), maps the
other's HBM state through CUDA IPC, and cross-shard CSQS run as direct
peer-memory segment exchanges (exchange_cross) between device-side barriers
(flags in the peer's memory; the host never waits). The reassembled state must
match the CPU ORACLE (the reference algorithm, simulator.py:179-235 for the
exchange) within 1e-10, the permutation exactly — in the default, lazy
(in place) and relabeled (double-buffered) layouts, where the optimizer's
SQS-CSQS-SQS sandwich costs one strided exchange. A second test runs the
33-qubit R=1 QFT/BV circuits as two 2^32-amplitude (64 GiB) in-place shards
and checks the analytic answer through the device-side fidelity.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CIRCUITS = [("example", 10, 4, 2, 8), ("random", 12, 5, 2, 6), ("random3", 13, 6, 3, 7),
            ("random18", 18, 8, 1, 10), ("random19r2", 19, 8, 2, 10), ("random19c12", 19, 12, 1, 12),
            # reference optimizer output, 2^23 per shard: specialised lazy passes and
            # the exchange overlapped with its neighbour passes
            ("qft24_c10_r1", 24, 10, 1, 23)]


def _circuit(name, n, c, r, seed=0):
    from conftest import EXAMPLE_OPTIMIZED
    if name == "example":
        return EXAMPLE_OPTIMIZED
    if name.startswith("qft"):
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        return open(os.path.join(root, "bench_circuits", name + ".txt")).read()
    from paper_2406_14084_b200 import LayoutParams, OptimizedCircuit, serialize_optimized
    from test_gpu_parity import _random_stream
    rng = np.random.default_rng(900 + n)
    ins = ()
    while not any(type(i).__name__ == "CrossRankSwap" for i in ins):
        ins = _random_stream(rng, n, r, c, 14)
    return serialize_optimized(OptimizedCircuit(n, LayoutParams(n=n, c=n - r, r=r), ins))


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_14084_b200.distributed import ShardedSimulator
        out = {}
        for name, n, c, r, b in CIRCUITS:
            text = _circuit(name, n, c, r)
            sim = ShardedSimulator(n, r, b=b, device=0)
            perm = sim.load_text(text, c if name.startswith("qft") else n - r)
            sim.reset()
            sim.run()
            shard = np.concatenate([sim.h.read(k, 0, 1 << (n - r)) for k in range(sim.count)])
            out[name] = (shard, sim.norm(), sim.logical_amplitudes(perm, 16), tuple(perm))
            del sim
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["default", "lazy", "relabel"])
def test_two_processes_share_the_state(gpu, mode):
    """`lazy`: the shards run in place with the lazy layout (QK_INPLACE, JIT at
    every size); `relabel`: double-buffered shards with relabeled stores. In
    both, cross-shard CSQS exchange strided segments of the current layout."""
    import torch.multiprocessing as mp
    from paper_2406_14084_b200 import LayoutParams, Simulator
    mgr = mp.Manager()
    results = mgr.dict()
    env = {"lazy": {"QK_INPLACE": "1", "QK_JIT": "0"}, "relabel": {"QK_JIT": "0"},
           "default": {"QK_OVERLAP": "1"}}.get(mode, {})
    os.environ.update(env)
    try:
        mp.spawn(_worker, args=(2, _port(), results), nprocs=2, join=True)
    finally:
        for k in env:
            os.environ.pop(k, None)
    from oracle import quokka_oracle as orc
    for name, n, c, r, b in CIRCUITS:
        text = _circuit(name, n, c, r)
        full, perm, _ = orc.simulate_text(text, n, n - r, r=r, b=b)
        got = np.concatenate([results[0][name][0], results[1][name][0]])
        assert np.max(np.abs(got - full)) <= 1e-10, name
        assert results[0][name][3] == perm, name
        assert abs(results[0][name][1] - np.linalg.norm(full)) <= 1e-12
        lidx = np.arange(16)
        src = np.zeros_like(lidx)
        for pos, q in enumerate(perm):
            src |= ((lidx >> q) & 1) << pos
        assert np.max(np.abs(results[1][name][2] - full[src])) <= 1e-10


def _big_worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), QK_INPLACE="1")
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_14084_b200.distributed import ShardedSimulator
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        out = {}
        for name in ("qft33_c10_r1", "bv33_c10_r1"):
            text = open(os.path.join(root, "bench_circuits", name + ".txt")).read()
            sim = ShardedSimulator(33, 1, device=0)
            perm = sim.load_text(text, 10)
            sim.reset()
            t = sim.run(perm)
            f = np.zeros((33, 2), dtype=np.complex128)
            if name.startswith("qft"):
                f[:] = 2 ** -0.5
            else:
                f[:, 0] = 1.0
            out[name] = (sim.fidelity_product(perm, f), sim.logical_amplitudes(perm, 4), t["xrs"],
                         tuple(sim.stats()))
            sim.close()
            del sim
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_two_processes_33_qubits_in_place(gpu):
    """Two processes x 2^32 amplitudes (64 GiB each, in place, one device):
    the reference optimizer's R=1 QFT33/BV33 streams with their CSQS as
    strided peer exchanges of 32 GiB per shard."""
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_big_worker, args=(2, _port(), results), nprocs=2, join=True)
    for name, amp0 in (("qft33_c10_r1", 2 ** -16.5), ("bv33_c10_r1", 1.0)):
        fid, amps, xrs, st = results[0][name]
        print(f"\n  {name}: 1-fidelity {1 - fid:.3e}, xrs {xrs:.4f} s, {st[8] / 2**30:.1f} GiB sent per shard")
        assert fid >= 1 - 1e-12, name
        assert abs(amps[0] - amp0) <= 1e-10
        assert results[1][name][0] == fid
