"""CPU, world_size 2 over gloo: the host logic of the multi-process CSQS.

Each process holds its shard of the global state (2^R ranks, `count` per
process), asks the native planner (qk_csqs_plan, no GPU) for its cross-shard
segment exchanges and in-shard pairs, executes them — the peer-memory swap of
the GPU path emulated with gloo send/recv — and the reassembled global vector
must equal the oracle's cross_rank_swap bit-exactly (simulator.py:179-235).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import quokka_oracle as orc

CASES = [
    # n, r, local_set, rank_set, b
    (8, 1, (6,), (7,), 7),
    (9, 2, (5, 6), (7, 8), 7),
    (9, 2, (6,), (8,), 3),
    (10, 3, None, None, 7),                 # S = 3: top three local bits <-> all rank bits
    (10, 3, (6,), (8,), 4),
    (10, 3, (4, 5, 6), (7, 8, 9), 7),
    (10, 3, (5, 6), (7, 9), 6),
    (11, 3, (7,), (10,), 8),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(rank, world, shard, segs_all):
    """Execute every rank's plan: the executor sends its slice and receives the peer's."""
    import torch
    for executor, segs in enumerate(segs_all):
        for my_off, peer, peer_off, length in segs:
            if rank == executor:
                out = torch.from_numpy(shard[my_off:my_off + length].view(np.float64).copy())
                dist.send(out, dst=peer)
                inc = torch.empty(2 * length, dtype=torch.float64)
                dist.recv(inc, src=peer)
                shard[my_off:my_off + length] = inc.numpy().view(np.complex128)
            elif rank == peer:
                inc = torch.empty(2 * length, dtype=torch.float64)
                dist.recv(inc, src=executor)
                out = torch.from_numpy(shard[peer_off:peer_off + length].view(np.float64).copy())
                dist.send(out, dst=executor)
                shard[peer_off:peer_off + length] = inc.numpy().view(np.complex128)


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_2406_14084_b200 import _lib
        ok = []
        for n, r, local_set, rank_set, b in CASES:
            L = n - r
            if rank_set is None:        # S = 3 case with the rank bits (7, 8, 9)
                local_set, rank_set = (L - 3, L - 2, L - 1), (L, L + 1, L + 2)
            count = (1 << r) // world
            nb = L + count.bit_length() - 1
            v = (np.arange(1 << n) + 0.5j * np.arange(1 << n)).astype(np.complex128)
            shard = v[rank << nb:(rank + 1) << nb].copy()
            segs, (in_a, in_b) = _lib.csqs_plan(n, r, count, rank, local_set, rank_set)
            segs_all = [None] * world
            dist.all_gather_object(segs_all, segs)
            _exchange(rank, world, shard, segs_all)
            if in_a:
                shard = orc.bitswap_permute(shard, in_a, in_b)   # the SQS kernel's job on the GPU
            parts = [torch.empty(2 << nb, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(shard.view(np.float64).copy()))
            got = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            size = 1 << L
            ref_parts = [v[q * size:(q + 1) * size].copy() for q in range(1 << r)]
            orc.cross_rank_swap(ref_parts, local_set, rank_set, n, r, b)
            ok.append(bool(np.array_equal(got, np.concatenate(ref_parts))))
        results[rank] = ok
    finally:
        dist.destroy_process_group()


def test_cross_shard_plan_world2():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert results[0] == results[1] == [True] * len(CASES), dict(results)


def test_plan_covers_each_pair_once():
    """Union over shards of the executed segments covers every off-diagonal
    segment pair exactly once (half each way)."""
    from paper_2406_14084_b200 import _lib
    n, r = 10, 3
    for count in (1, 2, 4):
        shards = (1 << r) // count
        moved = {}
        for sh in range(shards):
            segs, _ = _lib.csqs_plan(n, r, count, sh, (5, 6), (8, 9))
            for my_off, peer, peer_off, length in segs:
                for k in range(length):
                    a, bb = (sh, my_off + k), (peer, peer_off + k)
                    key = tuple(sorted((a, bb)))
                    moved[key] = moved.get(key, 0) + 1
        assert all(c == 1 for c in moved.values())
    with pytest.raises(ValueError):
        _lib.csqs_plan(n, r, 3, 0, (6,), (9,))
