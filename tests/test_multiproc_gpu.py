"""GPU, two processes sharing cuda:0: the multi-process shard path end to end.

Each process owns half of the 2^R rank partitions (qk_create_shard), maps the
other's HBM state through CUDA IPC, and cross-shard CSQS run as direct
peer-memory segment exchanges (exchange_cross) between host barriers (gloo).
Final state must equal the single-process simulation bit-for-bit in layout and
within 1e-12 in value (both run the same kernels on the same device).
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
            ("random18", 18, 8, 1, 10), ("random19r2", 19, 8, 2, 10), ("random19c12", 19, 12, 1, 12)]


def _circuit(name, n, c, r, seed=0):
    from conftest import EXAMPLE_OPTIMIZED
    if name == "example":
        return EXAMPLE_OPTIMIZED
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
            perm = sim.load_text(text, n - r)
            sim.reset()
            sim.run()
            shard = np.concatenate([sim.h.read(k, 0, 1 << (n - r)) for k in range(sim.count)])
            out[name] = (shard, sim.norm(), sim.logical_amplitudes(perm, 16))
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
    env = {"lazy": {"QK_INPLACE": "1", "QK_JIT": "0"}, "relabel": {"QK_JIT": "0"}}.get(mode, {})
    os.environ.update(env)
    try:
        mp.spawn(_worker, args=(2, _port(), results), nprocs=2, join=True)
    finally:
        for k in env:
            os.environ.pop(k, None)
    for name, n, c, r, b in CIRCUITS:
        text = _circuit(name, n, c, r)
        sim = Simulator(LayoutParams(n=n, c=n - r, r=r, b=b))
        perm = sim.load_text(text, n - r)
        res = sim.run_loaded(perm)
        full = res.physical_vector()
        got = np.concatenate([results[0][name][0], results[1][name][0]])
        assert np.max(np.abs(got - full)) <= 1e-12, name
        assert abs(results[0][name][1] - res.norm()) <= 1e-12
        assert np.max(np.abs(results[1][name][2] - res.logical_amplitudes(16))) <= 1e-12
