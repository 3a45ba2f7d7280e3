"""B200-native drop-in for the reference simulation module
(/root/reference/pkg/src/quokka/simulator.py).

Same names, signatures and error behaviour as the reference; the state lives in
HBM and every compute step runs in libqkb200.so (include/qkb200.h):

* `Simulator.run` loads the instruction stream once (native packing/compile)
  and replays it on the GPU (simulator.py:529-555).
* `StatePartition.amps` is a `DeviceAmps` view: a numpy-compatible window on a
  partition of the device state (reads/writes are D2H/H2D copies), so
  `res.partitions[0].amps[:2]`, `parts[0].amps[:] = v` and `np.abs(p.amps)`
  behave as with the reference's host arrays (simulator.py:43-46, 555).
* Kernel-level functions (`apply_gate_block`, `in_memory_swap`,
  `cross_rank_swap`, `apply_gate_full`) accept either device partitions or
  host numpy arrays; host arrays are staged through a device scratch state,
  the computation itself always runs on the GPU.

There is no CPU compute path: a missing library or GPU raises.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .circuit import LayoutParams, replay_permutation
from .errors import SimulationError

__all__ = ["SimulationError", "StatePartition", "SimConfig", "SimResult", "Simulator",
           "simulate", "init_state", "apply_gate_block", "in_memory_swap", "cross_rank_swap",
           "apply_gate_full", "get_amplitude", "bitswap", "bitshift", "shift_pairs",
           "DeviceAmps"]


# ---------------------------------------------------------------------------
# device-backed partitions


class DeviceAmps:
    """numpy-like view of partition `part` of a device state (2^L complex128)."""

    __array_priority__ = 100

    def __init__(self, handle: _lib.Handle, part: int):
        self._h = handle
        self._part = part
        self.size = 1 << handle.local
        self.shape = (self.size,)
        self.ndim = 1
        self.dtype = np.dtype(np.complex128)

    @property
    def handle(self) -> _lib.Handle:
        return self._h

    @property
    def part(self) -> int:
        return self._part

    def __len__(self) -> int:
        return self.size

    def __array__(self, dtype=None, copy=None):
        arr = self._h.read(self._part, 0, self.size)
        return arr if dtype is None else arr.astype(dtype)

    def copy(self) -> np.ndarray:
        return np.array(self)

    def _index(self, i) -> int:
        i = int(i)
        if i < 0:
            i += self.size
        if not 0 <= i < self.size:
            raise IndexError(f"index {i} out of range for size {self.size}")
        return i

    def __getitem__(self, key):
        if isinstance(key, (int, np.integer)):
            return complex(self._h.read(self._part, self._index(key), 1)[0])
        if isinstance(key, slice):
            start, stop, step = key.indices(self.size)
            if step == 1:
                return self._h.read(self._part, start, max(0, stop - start))
            return np.array(self)[key]
        idx = np.asarray(key)
        if idx.dtype == bool:
            return np.array(self)[idx]
        flat = np.where(idx < 0, idx + self.size, idx).astype(np.uint64).reshape(-1)
        base = (self._h.rank_lo + self._part) << self._h.local
        return self._h.gather(flat + np.uint64(base)).reshape(idx.shape)

    def __setitem__(self, key, value):
        if isinstance(key, (int, np.integer)):
            self._h.write(self._part, self._index(key), np.asarray([value], dtype=np.complex128))
            return
        if isinstance(key, slice):
            start, stop, step = key.indices(self.size)
            if step == 1:
                n = max(0, stop - start)
                vals = np.broadcast_to(np.asarray(value, dtype=np.complex128), (n,))
                self._h.write(self._part, start, np.ascontiguousarray(vals))
                return
        arr = np.array(self)
        arr[key] = value
        self._h.write(self._part, 0, arr)

    def __repr__(self):
        return f"DeviceAmps(part={self._part}, size={self.size})"


@dataclass
class StatePartition:                         # simulator.py:43-46
    rank_id: int
    amps: object


@dataclass
class SimConfig:                              # simulator.py:49-52
    layout: LayoutParams
    workers_per_rank: int = 1


def _device_list(layout: LayoutParams, device: int, devices):
    """Devices for a state: `devices` if given, else $QK_DEVICES (e.g. "0,1,2,3";
    an id may repeat), else None (one device; see _open_handle)."""
    import os
    if devices is None and os.environ.get("QK_DEVICES"):
        devices = [int(x) for x in os.environ["QK_DEVICES"].split(",") if x.strip()]
    return list(devices) if devices else None


def _open_handle(layout: LayoutParams, device: int = 0, devices=None) -> _lib.Handle:
    """One handle for the whole 2^N state. A state that does not fit `device`
    is split over the visible GPUs (largest power of two <= min(#GPUs, 2^R)),
    one host thread driving them all, like the reference's single-process
    Simulator over 2^R ranks (simulator.py:422-447)."""
    devs = _device_list(layout, device, devices)
    if devs and len(devs) > 1:
        return _lib.Handle(layout.n, layout.r, layout.b, devices=devs)
    try:
        return _lib.Handle(layout.n, layout.r, layout.b, devs[0] if devs else device)
    except SimulationError:
        ndev = min(_lib.device_count(), 1 << layout.r)
        k = 1 << (ndev.bit_length() - 1) if ndev > 0 else 0
        if devs or k < 2:
            raise
        return _lib.Handle(layout.n, layout.r, layout.b, devices=list(range(k)))


def init_state(layout: LayoutParams, device: int = 0, devices=None) -> list:
    """simulator.py:62-74 — |0...0> split across 2^R partitions, resident in HBM."""
    h = _open_handle(layout, device, devices)
    return [StatePartition(r, DeviceAmps(h, r)) for r in range(layout.num_ranks)]


# ---------------------------------------------------------------------------
# bit permutations (host index math, simulator.py:81-114)


def bitswap(i, a_bits, b_bits):
    """Exchange bit sorted(a)[k] with bit sorted(b)[k] of i (int or int array)."""
    if set(a_bits) & set(b_bits):
        raise ValueError("bit sets overlap")
    for x, y in zip(sorted(a_bits), sorted(b_bits)):
        flip = ((i >> x) ^ (i >> y)) & 1
        i = i ^ ((flip << x) | (flip << y))
    return i


def shift_pairs(a_bits, b_bits, cl: int, n_local: int):
    """simulator.py:91-106 — pairs compacting out-of-line partners above CL."""
    na = sum(1 for x in a_bits if x < cl)
    nb = sum(1 for x in b_bits if x < cl)
    d = abs(na - nb)
    if not d:
        return (), ()
    donors = b_bits if na > nb else a_bits
    far = sorted(x for x in donors if x >= cl)
    near = [x for x in range(cl, cl + d) if x < n_local]
    m = min(len(near), len(far))
    near, far = near[:m], far[:m]
    both = set(near) & set(far)
    return tuple(x for x in near if x not in both), tuple(x for x in far if x not in both)


def bitshift(t, a_bits, b_bits, cl: int, n_local: int):
    """simulator.py:109-114 — iteration-order bijection keeping the low CL bits."""
    p, q = shift_pairs(a_bits, b_bits, cl, n_local)
    return bitswap(t, p, q) if p else t


# ---------------------------------------------------------------------------
# kernel-level entry points (unit parity with the reference functions)

_scratch: dict = {}
_MAX_TILE = 13        # widest chunk one register-tiled block pass holds (qk_internal.h kMaxC)


def _scratch_handle(n: int, r: int = 0) -> _lib.Handle:
    key = (n, r)
    h = _scratch.get(key)
    if h is None:
        if len(_scratch) >= 4:          # bounded: each is a device state
            _scratch.clear()
        h = _lib.Handle(n, r, n - r)
        _scratch[key] = h
    return h


def _log2_size(amps) -> int:
    return int(len(amps)).bit_length() - 1


def apply_gate_block(partition: StatePartition, block, c: int, cl: int,
                     row_start: int = 0, row_stop: int | None = None) -> None:
    """simulator.py:338-357 — every gate of the block on rows of 2^c amplitudes."""
    words, params, npar = _lib.pack([block])
    amps = partition.amps
    rows = len(amps) >> c
    row_stop = rows if row_stop is None else row_stop
    if isinstance(amps, DeviceAmps):
        amps.handle.apply_block(amps.part, words, params, npar, c, row_start, row_stop)
        return
    h = _scratch_handle(_log2_size(amps))
    h.write(0, 0, amps)
    h.apply_block(0, words, params, npar, c, row_start, row_stop)
    amps[...] = h.read(0, 0, len(amps))


def apply_gate_full(amps, gate, part: int = 0, parts: int = 1) -> None:
    """simulator.py:360-376 — memory-level single gate: rows of
    2^(max target + 1) amplitudes, optionally only the aligned slice `part` of
    `parts` (units lo..hi, as the reference splits them). Runs as the device
    block pass over that row range (apply_gate_2d is the same gate on every row)."""
    n_local = _log2_size(amps)
    width = max(gate.targets) + 1
    if width > n_local:
        raise ValueError(f"gate target {max(gate.targets)} beyond {n_local} local qubits")
    n_units = len(amps) >> width
    if n_units >= parts > 1:
        lo, hi = n_units * part // parts, n_units * (part + 1) // parts
        if lo == hi:
            return
    else:
        if part != 0:
            return
        lo, hi = 0, n_units
    words, params, npar = _lib.pack([type("B", (), {"gates": (gate,)})()])
    if width <= _MAX_TILE:
        if isinstance(amps, DeviceAmps):
            amps.handle.apply_block(amps.part, words, params, npar, width, lo, hi)
            return
        h = _scratch_handle(n_local)
        h.write(0, 0, amps)
        h.apply_block(0, words, params, npar, width, lo, hi)
        amps[...] = h.read(0, 0, len(amps))
        return
    # wider than one tile: the memory-level device pass over each 2^width row
    unit = 1 << width
    h = _scratch_handle(width)
    for row in range(lo, hi):
        if isinstance(amps, DeviceAmps):
            h.write(0, 0, amps.handle.read(amps.part, row * unit, unit))
        else:
            h.write(0, 0, amps[row * unit:(row + 1) * unit])
        h.apply_gate_full(words, params, npar)
        out = h.read(0, 0, unit)
        if isinstance(amps, DeviceAmps):
            amps.handle.write(amps.part, row * unit, out)
        else:
            amps[row * unit:(row + 1) * unit] = out


def in_memory_swap(amps, out_set, in_set, cl: int, start: int = 0,
                   stop: int | None = None) -> None:
    """simulator.py:159-176 — new[i] = old[bitswap(i, out, in)], in place, bit-exact."""
    n_local = _log2_size(amps)
    for q in tuple(out_set) + tuple(in_set):
        if not (0 <= q < n_local):
            raise ValueError(f"swap bit {q} out of range for {n_local} local qubits")
    stop = (1 << n_local) if stop is None else stop
    if isinstance(amps, DeviceAmps):
        amps.handle.sqs(amps.part, out_set, in_set, cl, start, stop)
        return
    h = _scratch_handle(n_local)
    h.write(0, 0, amps)
    h.sqs(0, out_set, in_set, cl, start, stop)
    amps[...] = h.read(0, 0, len(amps))


def cross_rank_swap(partitions: list, local_set, rank_set, layout: LayoutParams,
                    buffers=None, run_tasks=None) -> None:
    """simulator.py:179-235 — swap top-of-local bits with rank bits across the
    2^R partitions (bit-exact; independent of B, which is only validated)."""
    amps0 = partitions[0].amps
    if (isinstance(amps0, DeviceAmps) and amps0.handle.count == len(partitions)
            and all(p.amps.handle is amps0.handle for p in partitions)):
        amps0.handle.csqs(local_set, rank_set)
        return
    h = _scratch_handle(layout.n, layout.r)
    if h.b != layout.b:
        h = _lib.Handle(layout.n, layout.r, layout.b)
    for k, p in enumerate(partitions):
        h.write(k, 0, np.asarray(p.amps))
    h.csqs(local_set, rank_set)
    for k, p in enumerate(partitions):
        p.amps[...] = h.read(k, 0, 1 << layout.local_qubits)


def get_amplitude(partitions: list, logical_index: int, permutation) -> complex:
    """simulator.py:410-419."""
    n = len(permutation)
    if not (0 <= logical_index < (1 << n)):
        raise IndexError(f"logical index {logical_index} out of range")
    phys = 0
    for pos in range(n):
        phys |= ((logical_index >> permutation[pos]) & 1) << pos
    local = _log2_size(partitions[0].amps)
    return complex(partitions[phys >> local].amps[phys & ((1 << local) - 1)])


# ---------------------------------------------------------------------------
# results and executor


def _shared_handle(partitions):
    a0 = partitions[0].amps if partitions else None
    if isinstance(a0, DeviceAmps) and a0.handle.count == len(partitions) and all(
            isinstance(p.amps, DeviceAmps) and p.amps.handle is a0.handle for p in partitions):
        return a0.handle
    return None


@dataclass
class SimResult:                              # simulator.py:383-407
    partitions: list
    final_permutation: tuple
    timings: dict = field(default_factory=dict)

    @property
    def layout_local(self) -> int:
        return _log2_size(self.partitions[0].amps)

    def norm(self) -> float:
        h = _shared_handle(self.partitions)
        if h is not None:
            return math.sqrt(h.sumsq())
        return math.sqrt(sum(float(np.sum(np.abs(np.asarray(p.amps)) ** 2))
                             for p in self.partitions))

    def physical_vector(self) -> np.ndarray:
        h = _shared_handle(self.partitions)
        if h is not None:
            return np.concatenate([h.read(k, 0, 1 << h.local) for k in range(h.count)])
        return np.concatenate([np.asarray(p.amps) for p in self.partitions])

    def logical_vector(self) -> np.ndarray:
        h = _shared_handle(self.partitions)
        n = len(self.final_permutation)
        if h is not None:
            return h.read_logical_range(self.final_permutation, 0, 1 << n)
        phys = self.physical_vector()
        idx = np.arange(1 << n, dtype=np.int64)
        src = np.zeros_like(idx)
        for pos, q in enumerate(self.final_permutation):
            src |= ((idx >> q) & 1) << pos
        return phys[src]

    def logical_amplitudes(self, count: int, start: int = 0) -> np.ndarray:
        """First `count` logical amplitudes (device gather; CLI --amps)."""
        h = _shared_handle(self.partitions)
        if h is None:
            return self.logical_vector()[start:start + count]
        return h.read_logical_range(self.final_permutation, start, count)

    def release(self) -> None:
        """Free the device state behind these partitions now (instead of at GC)."""
        h = _shared_handle(self.partitions)
        if h is not None:
            h.free()

    def fidelity_product(self, factors) -> float:
        """Normalised fidelity |<phi|psi>|^2 / (<phi|phi><psi|psi>) with the product
        state phi = (x)_q (f_q0|0> + f_q1|1>) over logical qubits (qk_overlap_product):
        one device read of the state, for analytic parity at any size."""
        h = _shared_handle(self.partitions)
        f = np.asarray(factors, dtype=np.complex128).reshape(-1, 2)
        if h is None:
            v = self.logical_vector()
            phi = np.ones(1, dtype=np.complex128)
            for q in range(f.shape[0]):
                phi = np.concatenate([phi * f[q, 0], phi * f[q, 1]])
            ov = np.vdot(phi, v)
        else:
            ov = h.overlap_product(self.final_permutation, f)
        nphi = float(np.prod(np.sum(np.abs(f) ** 2, axis=1)))
        return abs(ov) ** 2 / (nphi * self.norm() ** 2)

    def amplitude(self, logical_index: int) -> complex:
        h = _shared_handle(self.partitions)
        n = len(self.final_permutation)
        if h is not None:
            if not (0 <= logical_index < (1 << n)):
                raise IndexError(f"logical index {logical_index} out of range")
            return complex(h.read_logical(self.final_permutation, [logical_index])[0])
        return get_amplitude(self.partitions, logical_index, self.final_permutation)


class Simulator:
    """Executes optimized instruction streams on a B200 (simulator.py:422-569).

    All 2^R simulated ranks live contiguously in one HBM allocation, or, when
    the state does not fit one GPU (or `devices` / $QK_DEVICES name several),
    split over several GPUs driven by this one process (qk_create_multi;
    cross-GPU CSQS over NVLink peer memory). `workers_per_rank` is accepted for
    API parity and has no effect on the result (the reference guarantees
    bit-identical output for any value).
    """

    def __init__(self, layout: LayoutParams, workers_per_rank: int = 1, device: int = 0,
                 devices=None):
        self.layout = layout
        self.workers_per_rank = max(1, int(workers_per_rank))
        self._h = _open_handle(layout, device, devices)
        self.partitions = [StatePartition(r, DeviceAmps(self._h, r))
                           for r in range(layout.num_ranks)]
        self._program = None
        self.last_wall = 0.0

    @property
    def handle(self) -> _lib.Handle:
        return self._h

    def reset(self) -> None:                  # simulator.py:439-442
        self._h.reset()

    def close(self) -> None:                  # simulator.py:444-447
        """Like the reference, close() ends the executor but keeps the state
        readable: `simulate` closes the Simulator before returning a SimResult
        whose partitions alias it (simulator.py:555, 572-578). The device
        memory goes when the last view is dropped, or at once with release()."""

    def release(self) -> None:
        """Free the device state now (16 B x 2^N); every view of it becomes invalid."""
        self._h.free()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def total_workers(self) -> int:
        return self.layout.num_ranks * self.workers_per_rank

    def load(self, instructions) -> None:
        """Compile an instruction stream into device plans (cached by identity)."""
        if self._program is not None and self._program[0] is instructions:
            return
        words, params, npar = _lib.pack(instructions)
        self._h.load_packed(words, params, npar)
        self._program = (instructions,)

    def load_text(self, text: str, c: int | None = None) -> tuple:
        """Native parse + compile of the optimized text (the CLI path)."""
        self._h.load_text(text, self.layout.c if c is None else c)
        self._program = (object(),)
        return self._h.program_perm()

    def run_loaded(self, final_permutation) -> SimResult:
        timings, self.last_wall = self._h.run()
        return SimResult(self.partitions, tuple(final_permutation), timings)

    def run(self, opt, final_permutation=None) -> SimResult:   # simulator.py:529-555
        if hasattr(opt, "instructions"):
            if opt.num_qubits != self.layout.n:
                raise SimulationError(
                    f"circuit has {opt.num_qubits} qubits, layout has {self.layout.n}")
            instructions = opt.instructions
            final_permutation = opt.final_permutation
        else:
            instructions = tuple(opt)
            if final_permutation is None:
                final_permutation = replay_permutation(instructions, self.layout.n)
        self.load(instructions)
        return self.run_loaded(final_permutation)

    def run_gate_by_gate(self, raw) -> SimResult:  # simulator.py:557-569
        if self.layout.r != 0:
            raise SimulationError("gate-by-gate baseline runs on a single rank")
        block = type("GBGBlock", (), {"gates": tuple(raw.gates)})()
        words, params, npar = _lib.pack((block,))
        self._h.load_gate_by_gate(words, params, npar)
        self._program = None
        t0 = time.perf_counter()
        timings, _ = self._h.run()
        timings = {"gate": time.perf_counter() - t0 if not timings["gate"] else timings["gate"],
                   "ims": 0.0, "xrs": 0.0}
        return SimResult(self.partitions, tuple(range(self.layout.n)), timings)


def simulate(opt, cfg: SimConfig) -> SimResult:   # simulator.py:572-578
    sim = Simulator(cfg.layout, cfg.workers_per_rank)
    try:
        return sim.run(opt)
    finally:
        sim.close()
