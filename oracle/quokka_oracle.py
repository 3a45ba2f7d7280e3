"""CPU oracle for the all-in-cache (AIC) simulation path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference simulator
(`/root/reference/pkg/src/quokka/simulator.py`, `circuit.py`, `oracle.py`).
It exists to *check* the B200 product path, never to be it:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
  leg and `--impl reference` arm) may import it;
* the product package `paper_2406_14084_b200` never imports it and fails
  loudly when its CUDA library is missing.

Parity pin: `tests/golden/` holds vectors produced by the reference itself
(`oracle/gen_golden.py`, run in the build container where `/root/reference`
is importable); `tests/test_oracle_golden.py` checks this restatement against
every one of them (bit-exact for permutations, <=1e-12 for amplitudes).

Every function cites the reference file:line it restates. The structure is
the reference's algorithm (amplitude-major scratch batches per gate block,
pair walk with the m>n guard for in-memory swaps, windowed buffered
all-to-all for cross-rank swaps) so that timing it is a fair stand-in for
the reference CPU path.
"""
from __future__ import annotations

import cmath
import math
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# circuit.py:21, simulator.py:34 (0x3fe6a09e667f3bcc, one ULP below C's M_SQRT1_2)
DEFAULT_ANGLE = math.pi / 4
SQRT1_2 = 1.0 / math.sqrt(2.0)
BATCH_AMPS = 1 << 18          # simulator.py:35
SWAP_BATCH = 1 << 20          # simulator.py:36

# circuit.py:50-59 — arity / parameter count per kind ("D" is variable)
ARITY = {"H": 1, "X": 1, "U": 1, "RX": 1, "RY": 1, "RZ": 1,
         "CX": 2, "CP": 2, "SWAP": 2, "RZZ": 2}
NPARAMS = {"H": 0, "X": 0, "CX": 0, "SWAP": 0, "CP": 1, "RX": 1, "RY": 1,
           "RZ": 1, "RZZ": 1, "U": 3}


class OracleError(RuntimeError):
    pass


class OGate:
    """One gate: kind string, target tuple (targets[0] = matrix MSB), params."""
    __slots__ = ("kind", "targets", "gid", "params")

    def __init__(self, kind, targets, gid=0, params=()):
        self.kind = kind
        self.targets = tuple(int(t) for t in targets)
        self.gid = gid
        self.params = tuple(params)

    def __repr__(self):
        return f"OGate({self.kind},{self.targets})"


# ---------------------------------------------------------------------------
# text format (circuit.py:245-287 gate lines, :332-344 swap lines, :347-397 records)


def parse_optimized_text(text: str, n: int, c: int, local: int):
    """Return a list of ('B', [OGate]), ('S', out, in) and ('X', local, rank)."""
    rows = []
    for line in text.splitlines():
        body = line.split("#", 1)[0].split()
        if body:
            rows.append(body)
    out = []
    i = 0
    while i < len(rows):
        count = int(rows[i][0])
        payload = rows[i + 1:i + 1 + count]
        if len(payload) != count or count < 1:
            raise OracleError("bad record")
        head = payload[0][0]
        if head in ("SQS", "CSQS"):
            m = int(payload[0][1])
            ops = [int(t) for t in payload[0][2:]]
            a, b = tuple(ops[:m]), tuple(ops[m:])
            out.append(("S", a, b) if head == "SQS" else ("X", a, b))
        else:
            gates = []
            for toks in payload:
                kind = toks[0]
                if kind.startswith("D") and kind[1:].isdigit():
                    k = int(kind[1:])
                    tg = [int(t) for t in toks[1:1 + k]]
                    fl = [float(t) for t in toks[1 + k:]]
                    par = [complex(fl[2 * j], fl[2 * j + 1]) for j in range(1 << k)]
                    gates.append(OGate("D", tg, -1, par))
                else:
                    ar = ARITY[kind]
                    tg = [int(t) for t in toks[1:1 + ar]]
                    gid = int(toks[1 + ar])
                    par = [float(t) for t in toks[2 + ar:]] or [DEFAULT_ANGLE] * NPARAMS[kind]
                    gates.append(OGate(kind, tg, gid, par))
            out.append(("B", gates))
        i += 1 + count
    return out


def replay_permutation(instrs, n):
    """circuit.py:196-210 — physical position -> logical qubit after all swaps."""
    perm = list(range(n))
    for ins in instrs:
        if ins[0] in ("S", "X"):
            for pa, pb in zip(sorted(ins[1]), sorted(ins[2])):
                perm[pa], perm[pb] = perm[pb], perm[pa]
    return tuple(perm)


# ---------------------------------------------------------------------------
# gate matrices (circuit.py:420-463)


def gate_matrix(kind: str, params) -> np.ndarray:
    p = params
    if kind == "H":
        return np.array([[1, 1], [1, -1]], dtype=complex) * SQRT1_2
    if kind == "X":
        return np.array([[0, 1], [1, 0]], dtype=complex)
    if kind == "U":
        th, ph, lam = p
        ct, st = math.cos(th / 2), math.sin(th / 2)
        return np.array([[ct, -cmath.exp(1j * lam) * st],
                         [cmath.exp(1j * ph) * st, cmath.exp(1j * (ph + lam)) * ct]])
    if kind == "CX":
        return np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
    if kind == "CP":
        return np.diag([1, 1, 1, cmath.exp(1j * p[0])])
    if kind == "SWAP":
        return np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex)
    if kind == "RX":
        co, si = math.cos(p[0] / 2), math.sin(p[0] / 2)
        return np.array([[co, -1j * si], [-1j * si, co]])
    if kind == "RY":
        co, si = math.cos(p[0] / 2), math.sin(p[0] / 2)
        return np.array([[co, -si], [si, co]], dtype=complex)
    if kind == "RZ":
        return np.diag([cmath.exp(-1j * p[0] / 2), cmath.exp(1j * p[0] / 2)])
    if kind == "RZZ":
        em, ep = cmath.exp(-1j * p[0] / 2), cmath.exp(1j * p[0] / 2)
        return np.diag([em, ep, ep, em])
    if kind == "D":
        e = np.asarray(p, dtype=complex)
        if np.max(np.abs(np.abs(e) - 1.0)) > 1e-9:
            raise ValueError("non-unitary fused gate")
        return np.diag(e)
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# per-gate kernels over an amplitude-major scratch (2^width, tail)
# simulator.py:242-328


def _one_qubit(flat, g, tail):                       # simulator.py:242-264
    t = g.targets[0]
    v = flat.reshape(-1, 2, (1 << t) * tail)
    lo, hi = v[:, 0, :], v[:, 1, :]
    if g.kind == "H":
        s = (lo + hi) * SQRT1_2
        d = (lo - hi) * SQRT1_2
        lo[:] = s
        hi[:] = d
    elif g.kind == "X":
        keep = lo.copy()
        lo[:] = hi
        hi[:] = keep
    elif g.kind == "RZ":
        lo *= np.exp(-0.5j * g.params[0])
        hi *= np.exp(0.5j * g.params[0])
    else:
        m = gate_matrix(g.kind, g.params)
        n0 = m[0, 0] * lo + m[0, 1] * hi
        n1 = m[1, 0] * lo + m[1, 1] * hi
        lo[:] = n0
        hi[:] = n1


def _two_qubit(flat, g, tail):                       # simulator.py:267-299
    q0, q1 = g.targets
    lo, hi = min(q0, q1), max(q0, q1)
    v = flat.reshape(-1, 2, 1 << (hi - lo - 1), 2, (1 << lo) * tail)

    def quad(bh, bl):
        return v[:, bh, :, bl, :]

    if g.kind == "CX":                               # control = targets[0]
        a, b = (quad(1, 0), quad(1, 1)) if q0 == hi else (quad(0, 1), quad(1, 1))
        keep = a.copy()
        a[:] = b
        b[:] = keep
    elif g.kind == "SWAP":
        keep = quad(0, 1).copy()
        quad(0, 1)[:] = quad(1, 0)
        quad(1, 0)[:] = keep
    elif g.kind == "CP":
        quad(1, 1)[:] *= np.exp(1j * g.params[0])
    elif g.kind == "RZZ":
        em, ep = np.exp(-0.5j * g.params[0]), np.exp(0.5j * g.params[0])
        quad(0, 0)[:] *= em
        quad(1, 1)[:] *= em
        quad(0, 1)[:] *= ep
        quad(1, 0)[:] *= ep
    else:
        raise OracleError(f"no 2-qubit kernel for {g.kind}")


def diag_vector(g, width):                           # simulator.py:302-310
    entries = np.ascontiguousarray(np.diagonal(gate_matrix(g.kind, g.params)))
    k = len(g.targets)
    idx = np.arange(1 << width)
    sub = np.zeros(1 << width, dtype=np.int64)
    for j, q in enumerate(g.targets):                # targets[0] = table MSB
        sub |= ((idx >> q) & 1) << (k - 1 - j)
    return entries[sub]


def apply_gate_flat(flat, g, width, tail):           # simulator.py:313-328
    if any(t >= width for t in g.targets):
        raise OracleError(f"gate {g.kind} {g.targets} does not fit width {width}")
    if g.kind == "D":
        if tail == 1:
            flat.reshape(-1, 1 << width)[...] *= diag_vector(g, width)[None, :]
        else:
            flat.reshape(1 << width, tail)[...] *= diag_vector(g, width)[:, None]
    elif len(g.targets) == 1:
        _one_qubit(flat, g, tail)
    else:
        _two_qubit(flat, g, tail)


def apply_block_rows(amps, gates, c, row_start=0, row_stop=None):
    """simulator.py:338-357 — chunk batches copied amplitude-major, every gate
    applied in order, copied back."""
    view = amps.reshape(-1, 1 << c)
    row_stop = view.shape[0] if row_stop is None else row_stop
    step = max(1, BATCH_AMPS >> c)
    for r0 in range(row_start, row_stop, step):
        sub = view[r0:min(r0 + step, row_stop)]
        scratch = np.ascontiguousarray(sub.T)
        tail = scratch.shape[1]
        flat = scratch.reshape(-1)
        for g in gates:
            apply_gate_flat(flat, g, c, tail)
        sub[...] = scratch.T


def apply_gate_memory(amps, g, part=0, parts=1):    # simulator.py:331-376
    width = max(g.targets) + 1
    unit = 1 << width
    n_units = amps.size // unit
    if n_units >= parts > 1:
        lo, hi = n_units * part // parts, n_units * (part + 1) // parts
        if lo == hi:
            return
        sub = amps[lo * unit:hi * unit]
    else:
        if part != 0:
            return
        sub = amps
    arr = sub.reshape(-1, unit)
    step = max(1, BATCH_AMPS >> width)
    for r0 in range(0, arr.shape[0], step):
        apply_gate_flat(arr[r0:r0 + step].reshape(-1), g, width, 1)


# ---------------------------------------------------------------------------
# bit permutations (simulator.py:81-176)


def bitswap(i, a_bits, b_bits):                      # simulator.py:81-88
    if set(a_bits) & set(b_bits):
        raise ValueError("bit sets overlap")
    for a, b in zip(sorted(a_bits), sorted(b_bits)):
        d = ((i >> a) ^ (i >> b)) & 1
        i = i ^ (d << a) ^ (d << b)
    return i


def shift_pairs(a_bits, b_bits, cl, n_local):        # simulator.py:91-106
    a_in = [x for x in sorted(a_bits) if x < cl]
    b_in = [x for x in sorted(b_bits) if x < cl]
    d = abs(len(a_in) - len(b_in))
    if d == 0:
        return (), ()
    donors = b_bits if len(a_in) > len(b_in) else a_bits
    donor_out = sorted(x for x in donors if x >= cl)
    p0 = [x for x in range(cl, cl + d) if x < n_local]
    q0 = donor_out[:len(p0)]
    p0 = p0[:len(q0)]
    common = set(p0) & set(q0)
    return (tuple(x for x in p0 if x not in common),
            tuple(x for x in q0 if x not in common))


def bitshift(t, a_bits, b_bits, cl, n_local):        # simulator.py:109-114
    p, q = shift_pairs(a_bits, b_bits, cl, n_local)
    return bitswap(t, p, q) if p else t


def _pair_batches(n_local, a_bits, b_bits, cl, start, stop, batch=SWAP_BATCH):
    """simulator.py:117-148 — (m, n) batches over a 16-bit low/high split."""
    split = min(16, n_local)
    size = 1 << split
    lo_t = np.arange(size, dtype=np.int64)
    hi_t = np.arange(1 << max(0, n_local - split), dtype=np.int64) << split
    m_lo = bitshift(lo_t, a_bits, b_bits, cl, n_local)
    m_hi = bitshift(hi_t, a_bits, b_bits, cl, n_local)
    n_lo = bitswap(m_lo, a_bits, b_bits)
    n_hi = bitswap(m_hi, a_bits, b_bits)
    rows = max(1, batch // size)
    pos = start
    while pos < stop:
        if pos % size or stop - pos < size:
            h, o = pos >> split, pos & (size - 1)
            end = min(size, o + (stop - pos))
            yield m_hi[h] | m_lo[o:end], n_hi[h] | n_lo[o:end]
            pos += end - o
            continue
        h0 = pos >> split
        h1 = min(h0 + rows, stop >> split)
        yield ((m_hi[h0:h1, None] | m_lo[None, :]).reshape(-1),
               (n_hi[h0:h1, None] | n_lo[None, :]).reshape(-1))
        pos = h1 << split


def in_memory_swap(amps, out_set, in_set, cl=0, start=0, stop=None):
    """simulator.py:159-176 — new[i] = old[bitswap(i, out, in)] in place."""
    n_local = int(amps.size).bit_length() - 1
    for q in tuple(out_set) + tuple(in_set):
        if not (0 <= q < n_local):
            raise ValueError(f"swap bit {q} out of range for {n_local} local qubits")
    stop = (1 << n_local) if stop is None else stop
    for m, n in _pair_batches(n_local, out_set, in_set, cl, start, stop):
        sel = m > n
        mi, ni = m[sel], n[sel]
        keep = amps[mi]
        amps[mi] = amps[ni]
        amps[ni] = keep


def bitswap_permute(state, a_bits, b_bits):          # oracle.py:59-74
    idx = bitswap(np.arange(len(state), dtype=np.int64), tuple(a_bits), tuple(b_bits))
    return state[idx]


def cross_rank_swap(parts, local_set, rank_set, n, r, b, buffers=None, run=None):
    """simulator.py:179-235 — buffered in-place all-to-all in groups of 2^S
    ranks, one window of 2^(B-S) amplitudes per peer at a time."""
    local = n - r
    s = len(local_set)
    if tuple(sorted(local_set)) != tuple(range(local - s, local)):
        raise OracleError(f"cross-rank local set {local_set} is not top-of-local")
    if len(rank_set) != s:
        raise OracleError("cross-rank swap sets differ in size")
    for q in rank_set:
        if not (local <= q < n):
            raise OracleError(f"rank bit {q} outside [{local}, {n})")
    if b < s:
        raise OracleError(f"buffer of 2^{b} too small for {s} swap pairs")
    if buffers is None:
        buffers = [np.empty(1 << b, dtype=np.complex128) for _ in parts]
    if run is None:
        run = lambda tasks: [t() for t in tasks]
    seg = 1 << (local - s)
    win = 1 << (b - s)
    bitpos = sorted(q - local for q in rank_set)
    member, groups = {}, {}
    for rid in range(len(parts)):
        rho, key = 0, rid
        for k, bit in enumerate(bitpos):
            rho |= ((rid >> bit) & 1) << k
            key &= ~(1 << bit)
        member[rid] = rho
        groups.setdefault(key, [None] * (1 << s))[rho] = rid

    def send(rid, members, off, w):
        def task():
            x = member[rid]
            for y, peer in enumerate(members):
                buffers[peer][x * win:x * win + w] = parts[rid][y * seg + off:y * seg + off + w]
        return task

    def recv(rid, off, w):
        def task():
            for x in range(1 << s):
                parts[rid][x * seg + off:x * seg + off + w] = buffers[rid][x * win:x * win + w]
        return task

    for off in range(0, seg, win):
        w = min(win, seg - off)
        run([send(rid, mem, off, w) for mem in groups.values() for rid in mem])
        run([recv(rid, off, w) for mem in groups.values() for rid in mem])


# ---------------------------------------------------------------------------
# readback (simulator.py:393-419, oracle.py:149-160)


def logical_indices_to_physical(idx, perm):
    idx = np.asarray(idx, dtype=np.int64)
    phys = np.zeros_like(idx)
    for pos in range(len(perm)):
        phys |= ((idx >> perm[pos]) & 1) << pos
    return phys


def logical_state(physical, perm):
    n = len(perm)
    return physical[logical_indices_to_physical(np.arange(1 << n, dtype=np.int64), perm)]


def norm(parts):
    return math.sqrt(sum(float(np.sum(np.abs(p) ** 2)) for p in parts))


# ---------------------------------------------------------------------------
# executor (simulator.py:422-569)


class OracleSimulator:
    """CPU restatement of `Simulator`: 2^R partitions, per-class wall timings."""

    def __init__(self, n, c, r=0, cl=2, b=None, workers=1):
        self.n, self.c, self.r = n, c, r
        self.cl = min(cl, c)
        self.local = n - r
        self.b = self.local if b is None else b
        self.workers = max(1, workers)
        self.parts = [np.zeros(1 << self.local, dtype=np.complex128) for _ in range(1 << r)]
        self.parts[0][0] = 1.0
        self._pool = None
        self._buffers = None

    def close(self):
        if self._pool is not None:
            self._pool.shutdown()
            self._pool = None

    def _run(self, tasks):                           # simulator.py:459-471
        tasks = list(tasks)
        total = len(self.parts) * self.workers
        if total == 1 or len(tasks) == 1 or self.n < 18:
            for t in tasks:
                t()
            return
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=total)
        for f in [self._pool.submit(t) for t in tasks]:
            f.result()

    def block(self, gates, rows=None):               # simulator.py:481-511
        chunked = all(t < self.c for g in gates for t in g.targets)
        if chunked:
            nrows = 1 << (self.local - self.c) if rows is None else rows
            w = min(self.workers, nrows)
            self._run([(lambda p=p, a=nrows * i // w, z=nrows * (i + 1) // w:
                        apply_block_rows(p, gates, self.c, a, z))
                       for p in self.parts for i in range(w)])
            return
        for g in gates:
            if max(g.targets) >= self.local:
                raise OracleError(f"gate target {max(g.targets)} beyond local range")
        for g in gates:
            self._run([(lambda p=p, i=i, g=g: apply_gate_memory(p, g, i, self.workers))
                       for p in self.parts for i in range(self.workers)])

    def sqs(self, out_set, in_set, start=0, stop=None):   # simulator.py:513-523
        size = 1 << self.local if stop is None else stop - start
        w = min(self.workers, max(1, size // SWAP_BATCH)) or 1
        self._run([(lambda p=p, a=start + size * i // w, z=start + size * (i + 1) // w:
                     in_memory_swap(p, out_set, in_set, self.cl, a, z))
                   for p in self.parts for i in range(w)])

    def csqs(self, local_set, rank_set):             # simulator.py:525-527
        if self._buffers is None:
            self._buffers = [np.empty(1 << self.b, dtype=np.complex128) for _ in self.parts]
        cross_rank_swap(self.parts, local_set, rank_set, self.n, self.r, self.b,
                        self._buffers, self._run)

    def run(self, instrs):                           # simulator.py:529-555
        timings = {"gate": 0.0, "ims": 0.0, "xrs": 0.0}
        for ins in instrs:
            t0 = time.perf_counter()
            if ins[0] == "B":
                self.block(ins[1])
                timings["gate"] += time.perf_counter() - t0
            elif ins[0] == "S":
                self.sqs(ins[1], ins[2])
                timings["ims"] += time.perf_counter() - t0
            else:
                self.csqs(ins[1], ins[2])
                timings["xrs"] += time.perf_counter() - t0
        return timings

    def physical(self):
        return np.concatenate(self.parts)


def simulate_text(text, n, c, r=0, b=None, cl=2, workers=1):
    """Parse + run from |0..0>; returns (physical vector, final permutation, timings)."""
    local = n - r
    instrs = parse_optimized_text(text, n, c, local)
    sim = OracleSimulator(n, c, r, cl, b, workers)
    try:
        t = sim.run(instrs)
    finally:
        sim.close()
    return sim.physical(), replay_permutation(instrs, n), t


def dense_apply(state, g, n):                        # oracle.py:29-43
    mat = gate_matrix(g.kind, g.params)
    k = len(g.targets)
    tensor = state.reshape([2] * n)
    axes = [n - 1 - q for q in g.targets]
    rest = [a for a in range(n) if a not in axes]
    tensor = np.transpose(tensor, axes + rest).reshape(1 << k, -1)
    tensor = (mat @ tensor).reshape([2] * n)
    return np.transpose(tensor, np.argsort(axes + rest)).reshape(-1)
