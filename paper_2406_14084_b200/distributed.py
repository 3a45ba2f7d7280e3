"""One process per GPU: the 2^R rank partitions of the state are sharded over
the processes of a torch.distributed job (rank = top R bits,
circuit.py:157-163). Gate blocks and SQS are shard-local; a CSQS whose rank
bits cross shards is a peer-to-peer segment exchange over NVLink: every shard
maps its peers' HBM state through CUDA IPC (qk_ipc_handle / qk_ipc_open) and
the swap kernel reads and writes peer memory directly
(qk_runtime.cpp: csqs_plan / exchange_cross). The shards of an exchange meet
on flags in each other's memory (a device-side barrier on the stream), so the
host never waits inside a run. torch.distributed is plumbing only: the IPC
handle all-gather and the cross-shard reductions of the readback. (The host
barrier callback is registered too; it only runs under QK_HOST_BARRIER=1.)
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .circuit import replay_permutation


def _device_uuid(dev: int) -> str:
    try:
        import torch
        return str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:  # noqa: BLE001 — unknown: treat every shard as its own GPU
        import os
        return f"{os.getpid()}:{dev}"


class ShardedSimulator:
    """Shard of a 2^R-rank state held by this process (count = 2^R / world)."""

    def __init__(self, n: int, r: int, b: int | None = None, device: int | None = None,
                 group=None):
        import torch.distributed as dist
        self._dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world & (self.world - 1) or self.world > (1 << r):
            raise ValueError(f"world size {self.world} must be a power of two <= 2^R = {1 << r}")
        self.n, self.r = n, r
        self.b = n - r if b is None else b
        self.count = (1 << r) // self.world
        dev = self.rank if device is None else device
        self.h = _lib.Handle(n, r, self.b, dev, rank_lo=self.rank * self.count, count=self.count)
        # map every peer's state (CUDA IPC over NVLink)
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.lib().qk_ipc_handle(self.h.ptr, buf))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(buf.raw), group=group)
        for peer, hb in enumerate(handles):
            if peer != self.rank:
                raw = ctypes.create_string_buffer(hb, 128)
                _lib.check(_lib.lib().qk_ipc_open(self.h.ptr, peer, raw))
        self._cb = _lib.BARRIER_FN(self._barrier)
        _lib.check(_lib.lib().qk_set_barrier(self.h.ptr, self._cb, None))
        # pipeline the exchanges with the neighbour passes when every shard has
        # its own GPU (NVLink transfer next to HBM passes; shards sharing one
        # GPU would share its HBM)
        uuids = [None] * self.world
        dist.all_gather_object(uuids, _device_uuid(dev), group=group)
        _lib.check(_lib.lib().qk_set_overlap(self.h.ptr, int(len(set(uuids)) == self.world)))
        self.perm = tuple(range(n))

    def close(self) -> None:
        """Free this shard's state now. Collective: a peer's memory is only
        released once every shard has closed its IPC mapping of it, so the
        shards must all close before any of them allocates again."""
        self.h.free()
        self._dist.barrier(group=self.group)

    def _barrier(self, _ctx) -> int:
        try:
            self._dist.barrier(group=self.group)
            return 0
        except Exception:  # noqa: BLE001 — reported to the C side as a failed barrier
            return 1

    # -- program ------------------------------------------------------------

    def load_text(self, text: str, c: int) -> tuple:
        self.h.load_text(text, c)
        self.perm = self.h.program_perm()
        return self.perm

    def load(self, instructions) -> tuple:
        words, params, npar = _lib.pack(instructions)
        self.h.load_packed(words, params, npar)
        self.perm = replay_permutation(instructions, self.n)
        return self.perm

    def reset(self) -> None:
        self.h.reset()

    def run(self, perm=None) -> dict:
        timings, _ = self.h.run()
        return timings

    def sync(self) -> None:
        self.h.sync()

    def stats(self, reset: bool = False):
        return self.h.stats(reset)

    # -- readback -----------------------------------------------------------

    def _allreduce(self, arr: np.ndarray) -> np.ndarray:
        import torch
        t = torch.from_numpy(np.ascontiguousarray(arr))
        backend = self._dist.get_backend(self.group)
        if backend == "nccl":
            t = t.cuda()
        self._dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def norm(self) -> float:
        return math.sqrt(float(self._allreduce(np.array([self.h.sumsq()]))[0]))

    def overlap_product(self, perm, factors) -> complex:
        """<phi|psi> with a product state over logical qubits (qk_overlap_product),
        summed over the shards."""
        part = self.h.overlap_product(perm, factors)
        tot = self._allreduce(np.array([part.real, part.imag]))
        return complex(tot[0], tot[1])

    def fidelity_product(self, perm, factors) -> float:
        """Normalised fidelity with the product state (see SimResult.fidelity_product)."""
        f = np.asarray(factors, dtype=np.complex128).reshape(-1, 2)
        nphi = float(np.prod(np.sum(np.abs(f) ** 2, axis=1)))
        return abs(self.overlap_product(perm, f)) ** 2 / (nphi * self.norm() ** 2)

    def logical_amplitudes(self, perm, count: int, start: int = 0) -> np.ndarray:
        """First `count` logical amplitudes (simulator.py:410-419), gathered on
        their owning shard and summed across shards."""
        idx = np.arange(start, start + count, dtype=np.int64)
        phys = np.zeros_like(idx)
        for pos, q in enumerate(perm):
            phys |= ((idx >> q) & 1) << pos
        nb = self.n - self.r + int(self.count).bit_length() - 1
        owner = phys >> nb
        mine = owner == self.rank
        out = np.zeros(count, dtype=np.complex128)
        if mine.any():
            out[mine] = self.h.gather(phys[mine].astype(np.uint64))
        return self._allreduce(out.view(np.float64)).view(np.complex128)
