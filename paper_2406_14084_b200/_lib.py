"""ctypes binding of the C ABI in include/qkb200.h (libqkb200.so, built in-tree).

There is no fallback: if the shared library is missing the import of any
compute entry point raises. Build it with
`python -c "import __graft_entry__ as g; g.build()"`.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import CudaError, ParseError, SimulationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# QK_LIB_PATH: dev A/B runs against another build of the same library
LIB_PATH = os.environ.get("QK_LIB_PATH") or os.path.join(_HERE, "libqkb200.so")

QK_OK, QK_EINVAL, QK_EPARSE, QK_ESIM, QK_ENOMEM, QK_ECUDA = 0, -1, -2, -3, -4, -5
INS_BLOCK, INS_SQS, INS_CSQS = 0, 1, 2
KIND_CODE = {"H": 0, "X": 1, "U": 2, "CX": 3, "CP": 4, "SWAP": 5, "RX": 6, "RY": 7,
             "RZ": 8, "RZZ": 9, "D": 10}
CODE_KIND = {v: k for k, v in KIND_CODE.items()}

_lib = None
_lock = threading.Lock()

c_int, c_int32, c_size, c_u64, c_dbl, c_void = (ctypes.c_int, ctypes.c_int32, ctypes.c_size_t,
                                               ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p)
P = ctypes.POINTER
BARRIER_FN = ctypes.CFUNCTYPE(c_int, c_void)

_SIGS = {
    "qk_version": (c_int, []),
    "qk_jit_available": (c_int, []),
    "qk_last_error": (ctypes.c_char_p, []),
    "qk_device_count": (c_int, [P(c_int)]),
    "qk_create": (c_int, [c_int, c_int, c_int, c_int, P(c_void)]),
    "qk_create_shard": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, P(c_void)]),
    "qk_create_multi": (c_int, [c_int, c_int, c_int, P(c_int), c_int, P(c_void)]),
    "qk_destroy": (c_int, [c_void]),
    "qk_reset": (c_int, [c_void]),
    "qk_layout": (c_int, [c_void, P(c_int), P(c_int), P(c_int), P(c_int), P(c_int)]),
    "qk_load_text": (c_int, [c_void, ctypes.c_char_p, c_size, c_int, P(c_int)]),
    "qk_parse_text": (c_int, [ctypes.c_char_p, c_size, c_int, c_int, c_int, P(c_int32), P(c_size),
                              P(c_dbl), P(c_size), P(c_int)]),
    "qk_load_packed": (c_int, [c_void, P(c_int32), c_size, P(c_dbl), c_size]),
    "qk_plan_dry": (c_int, [ctypes.c_char_p, c_size, c_int, c_int, c_int, ctypes.c_char_p, P(c_int)]),
    "qk_reblock_packed": (c_int, [P(c_int32), c_size, P(c_dbl), c_size, c_int, c_int, P(c_int32),
                                  P(c_size), P(c_dbl), P(c_size), P(c_int32), P(c_int)]),
    "qk_reblock_shard": (c_int, [P(c_int32), c_size, P(c_dbl), c_size, c_int, c_int, c_int, P(c_int32),
                                 P(c_size), P(c_dbl), P(c_size), P(c_int32), P(c_int)]),
    "qk_load_gate_by_gate": (c_int, [c_void, P(c_int32), c_size, P(c_dbl), c_size]),
    "qk_program_info": (c_int, [c_void, P(c_int), P(c_int), P(c_int), P(c_int), P(c_int32)]),
    "qk_run": (c_int, [c_void, P(c_dbl)]),
    "qk_kernel_stats": (c_int, [c_void, P(c_dbl), c_int]),
    "qk_set_profiling": (c_int, [c_void, c_int]),
    "qk_sumsq": (c_int, [c_void, P(c_dbl)]),
    "qk_read_physical": (c_int, [c_void, c_int, c_u64, c_u64, P(c_dbl)]),
    "qk_write_physical": (c_int, [c_void, c_int, c_u64, c_u64, P(c_dbl)]),
    "qk_gather": (c_int, [c_void, P(c_u64), c_u64, P(c_dbl)]),
    "qk_read_logical": (c_int, [c_void, P(c_int32), P(c_u64), c_u64, P(c_dbl)]),
    "qk_read_logical_range": (c_int, [c_void, P(c_int32), c_u64, c_u64, P(c_dbl)]),
    "qk_overlap_product": (c_int, [c_void, P(c_int32), P(c_dbl), P(c_dbl)]),
    "qk_apply_block": (c_int, [c_void, c_int, P(c_int32), c_size, P(c_dbl), c_size, c_int, c_u64,
                               c_u64]),
    "qk_sqs": (c_int, [c_void, c_int, P(c_int32), P(c_int32), c_int, c_int, c_u64, c_u64]),
    "qk_csqs": (c_int, [c_void, P(c_int32), P(c_int32), c_int]),
    "qk_apply_gate_full": (c_int, [c_void, P(c_int32), c_size, P(c_dbl), c_size]),
    "qk_ipc_handle": (c_int, [c_void, c_void]),
    "qk_csqs_plan": (c_int, [c_int, c_int, c_int, c_int, P(c_int32), P(c_int32), c_int, P(c_u64),
                             P(c_size), P(c_int32), P(c_int)]),
    "qk_ipc_open": (c_int, [c_void, c_int, c_void]),
    "qk_set_barrier": (c_int, [c_void, BARRIER_FN, c_void]),
    "qk_set_overlap": (c_int, [c_void, c_int]),
    "qk_mark": (c_int, [c_void, c_int]),
    "qk_mark_elapsed": (c_int, [c_void, c_int, c_int, P(c_dbl)]),
    "qk_sync": (c_int, [c_void]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load libqkb200.so once; raise loudly when it is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"native library {LIB_PATH} is missing; build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().qk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, err_line: int = 0) -> None:
    if rc == QK_OK:
        return
    msg = last_error()
    if rc == QK_EINVAL:
        raise ValueError(msg)
    if rc == QK_EPARSE:
        body = msg.split(": ", 1)[1] if msg.startswith("line ") and ": " in msg else msg
        raise ParseError(err_line or _line_of(msg), body)
    if rc in (QK_ESIM, QK_ENOMEM):
        raise SimulationError(msg)
    raise CudaError(msg or f"native error {rc}")


def _line_of(msg: str) -> int:
    try:
        return int(msg.split(":", 1)[0].split()[1])
    except (IndexError, ValueError):
        return 0


def dptr(a: np.ndarray):
    return a.ctypes.data_as(P(c_dbl))


def iptr(a: np.ndarray):
    return a.ctypes.data_as(P(c_int32))


def uptr(a: np.ndarray):
    return a.ctypes.data_as(P(c_u64))


def jit_available() -> bool:
    """NVRTC present: large-state passes are specialised at load (qk_jit_available)."""
    return bool(lib().qk_jit_available())


def device_count() -> int:
    n = c_int(0)
    rc = lib().qk_device_count(ctypes.byref(n))
    return n.value if rc == QK_OK else 0


# ---------------------------------------------------------------------------
# packing of instruction objects (duck-typed: ours or the reference's)


def kind_name(kind) -> str:
    return kind.value if hasattr(kind, "value") else str(kind)


def pack(instructions):
    """GateBlock / InMemSwap / CrossRankSwap objects -> (int32 words, float64 params)."""
    words: list[int] = []
    params: list[float] = []
    for ins in instructions:
        if hasattr(ins, "gates"):
            words += [INS_BLOCK, len(ins.gates)]
            for g in ins.gates:
                kn = kind_name(g.kind)
                words += [KIND_CODE[kn], len(g.targets), *[int(t) for t in g.targets]]
                if kn == "D":
                    flat = []
                    for e in g.params:
                        e = complex(e)
                        flat += [e.real, e.imag]
                else:
                    flat = [float(x) for x in g.params]
                words.append(len(flat))
                params += flat
        elif hasattr(ins, "out_set"):
            words += [INS_SQS, len(ins.out_set), *map(int, ins.out_set), *map(int, ins.in_set)]
        elif hasattr(ins, "local_set"):
            words += [INS_CSQS, len(ins.local_set), *map(int, ins.local_set), *map(int, ins.rank_set)]
        else:
            raise TypeError(f"unknown instruction {ins!r}")
    return (np.ascontiguousarray(words, dtype=np.int32),
            np.ascontiguousarray(params if params else [0.0], dtype=np.float64)[:max(1, len(params))],
            len(params))


def parse_text(text: str, n: int, local: int, c: int):
    """Native parse (circuit.py:347-397) -> (words, params, gate ids)."""
    L = lib()
    raw = text.encode()
    nw, npar, line = c_size(0), c_size(0), c_int(0)
    rc = L.qk_parse_text(raw, len(raw), n, local, c, None, ctypes.byref(nw), None,
                         ctypes.byref(npar), ctypes.byref(line))
    check(rc, line.value)
    words = np.zeros(max(1, nw.value), dtype=np.int32)
    params = np.zeros(max(1, npar.value), dtype=np.float64)
    rc = L.qk_parse_text(raw, len(raw), n, local, c, iptr(words), ctypes.byref(nw), dptr(params),
                         ctypes.byref(npar), ctypes.byref(line))
    check(rc, line.value)
    return words[:nw.value], params[:npar.value]


def plan_dry(text: str, n: int, c: int, second_buffer: bool = True, dump_dir: str | None = None) -> int:
    """Host-only plan of a circuit (qk_plan_dry) -> number of passes."""
    raw = text.encode()
    npass = c_int(0)
    check(lib().qk_plan_dry(raw, len(raw), n, c, int(second_buffer),
                            dump_dir.encode() if dump_dir else None, ctypes.byref(npass)))
    return npass.value


def reblock_packed(words, params, n: int, cap: int, nlocal: int | None = None):
    """Cross-block pass schedule (qk_reblock_packed, or qk_reblock_shard for a
    shard of `nlocal` local bits) -> (words, params, p2w, npass); npass 0 when
    the program cannot be rescheduled."""
    L = lib()
    w = np.ascontiguousarray(words, dtype=np.int32)
    p = np.ascontiguousarray(params, dtype=np.float64)
    if p.size == 0:
        p = np.zeros(1)

    def call(ow, nw, op, npar, p2w, npass):
        if nlocal is None:
            return L.qk_reblock_packed(iptr(w), w.size, dptr(p), p.size, n, cap, ow, nw, op, npar, p2w, npass)
        return L.qk_reblock_shard(iptr(w), w.size, dptr(p), p.size, n, nlocal, cap, ow, nw, op, npar, p2w, npass)

    nw, npar, npass = c_size(0), c_size(0), c_int(0)
    check(call(None, ctypes.byref(nw), None, ctypes.byref(npar), None, ctypes.byref(npass)))
    if npass.value == 0:
        return None, None, None, 0
    ow = np.zeros(max(1, nw.value), dtype=np.int32)
    op = np.zeros(max(1, npar.value), dtype=np.float64)
    p2w = np.zeros(n, dtype=np.int32)
    check(call(iptr(ow), ctypes.byref(nw), dptr(op), ctypes.byref(npar), iptr(p2w), ctypes.byref(npass)))
    return ow[:nw.value], op[:npar.value], p2w, npass.value


def csqs_plan(n: int, r: int, count: int, shard: int, local_set, rank_set):
    """Cross-shard exchange plan -> (segments [(my_off, peer, peer_off, len)], in-shard pairs)."""
    a = np.ascontiguousarray(local_set, dtype=np.int32)
    b = np.ascontiguousarray(rank_set, dtype=np.int32)
    nseg, nloc = c_size(0), c_int(0)
    check(lib().qk_csqs_plan(n, r, count, shard, iptr(a), iptr(b), len(a), None, ctypes.byref(nseg),
                             None, ctypes.byref(nloc)))
    segs = np.zeros(max(1, 4 * nseg.value), dtype=np.uint64)
    pairs = np.zeros(max(1, 2 * nloc.value), dtype=np.int32)
    check(lib().qk_csqs_plan(n, r, count, shard, iptr(a), iptr(b), len(a), uptr(segs),
                             ctypes.byref(nseg), iptr(pairs), ctypes.byref(nloc)))
    seg_list = [tuple(int(x) for x in segs[4 * i:4 * i + 4]) for i in range(nseg.value)]
    m = nloc.value
    return seg_list, (tuple(int(x) for x in pairs[:m]), tuple(int(x) for x in pairs[m:2 * m]))


class Handle:
    """Owner of one qk_sim*; frees the device state when garbage collected."""

    def __init__(self, n: int, r: int, b: int, device: int = 0, rank_lo: int = 0, count: int = 0,
                 devices=None):
        self.ptr = c_void(None)
        L = lib()
        self.devices = tuple(devices) if devices else (device,)
        if devices and len(devices) > 1:
            devs = (c_int * len(devices))(*devices)
            check(L.qk_create_multi(n, r, b, devs, len(devices), ctypes.byref(self.ptr)))
        elif count:
            check(L.qk_create_shard(n, r, b, device, rank_lo, count, ctypes.byref(self.ptr)))
        else:
            check(L.qk_create(n, r, b, device, ctypes.byref(self.ptr)))
        self.n, self.r, self.b, self.device = n, r, b, self.devices[0]
        self.rank_lo = rank_lo
        self.count = count or (1 << r)
        self.local = n - r
        self.program_key = None
        self._keep = None

    def __del__(self):
        self.free()

    def free(self):
        """Destroy the native handle (device state and plans) now."""
        if getattr(self, "ptr", None) and self.ptr.value and _lib is not None:
            _lib.qk_destroy(self.ptr)
            self.ptr = c_void(None)

    def reset(self):
        check(lib().qk_reset(self.ptr))

    def load_packed(self, words, params, nparams):
        check(lib().qk_load_packed(self.ptr, iptr(words), len(words), dptr(params), nparams))

    def load_gate_by_gate(self, words, params, nparams):
        check(lib().qk_load_gate_by_gate(self.ptr, iptr(words), len(words), dptr(params), nparams))

    def load_text(self, text: str, c: int):
        raw = text.encode()
        ni = c_int(0)
        check(lib().qk_load_text(self.ptr, raw, len(raw), c, ctypes.byref(ni)))
        return ni.value

    def program_perm(self):
        perm = np.zeros(self.n, dtype=np.int32)
        check(lib().qk_program_info(self.ptr, None, None, None, None, iptr(perm)))
        return tuple(int(x) for x in perm)

    def run(self):
        t = np.zeros(4, dtype=np.float64)
        check(lib().qk_run(self.ptr, dptr(t)))
        return {"gate": float(t[0]), "ims": float(t[1]), "xrs": float(t[2])}, float(t[3])

    def stats(self, reset=False):
        out = np.zeros(16, dtype=np.float64)
        check(lib().qk_kernel_stats(self.ptr, dptr(out), int(reset)))
        return out

    def sumsq(self) -> float:
        v = c_dbl(0.0)
        check(lib().qk_sumsq(self.ptr, ctypes.byref(v)))
        return v.value

    def read(self, part: int, off: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.complex128)
        if count:
            check(lib().qk_read_physical(self.ptr, part, off, count, out.ctypes.data_as(P(c_dbl))))
        return out

    def write(self, part: int, off: int, values) -> None:
        vals = np.ascontiguousarray(values, dtype=np.complex128)
        if vals.size:
            check(lib().qk_write_physical(self.ptr, part, off, vals.size,
                                          vals.ctypes.data_as(P(c_dbl))))

    def gather(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.empty(idx.size, dtype=np.complex128)
        if idx.size:
            check(lib().qk_gather(self.ptr, uptr(idx), idx.size, out.ctypes.data_as(P(c_dbl))))
        return out

    def read_logical(self, perm, idx) -> np.ndarray:
        pm = np.ascontiguousarray(perm, dtype=np.int32)
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.empty(idx.size, dtype=np.complex128)
        if idx.size:
            check(lib().qk_read_logical(self.ptr, iptr(pm), uptr(idx), idx.size,
                                        out.ctypes.data_as(P(c_dbl))))
        return out

    def read_logical_range(self, perm, start: int, count: int) -> np.ndarray:
        pm = np.ascontiguousarray(perm, dtype=np.int32)
        out = np.empty(count, dtype=np.complex128)
        if count:
            check(lib().qk_read_logical_range(self.ptr, iptr(pm), start, count,
                                              out.ctypes.data_as(P(c_dbl))))
        return out

    def overlap_product(self, perm, factors) -> complex:
        """<phi|psi> with the product state phi = (x)_q (f_q0|0> + f_q1|1>) over
        logical qubits; factors is (n, 2) complex (qk_overlap_product)."""
        pm = np.ascontiguousarray(perm if perm is not None else range(self.n), dtype=np.int32)
        f = np.ascontiguousarray(np.asarray(factors, dtype=np.complex128).reshape(self.n, 2))
        out = np.zeros(2, dtype=np.float64)
        check(lib().qk_overlap_product(self.ptr, iptr(pm), f.view(np.float64).ctypes.data_as(P(c_dbl)),
                                       dptr(out)))
        return complex(out[0], out[1])

    def apply_block(self, part, words, params, nparams, c, row_start, row_stop):
        check(lib().qk_apply_block(self.ptr, part, iptr(words), len(words), dptr(params), nparams,
                                   c, row_start, row_stop))

    def apply_gate_full(self, words, params, nparams):
        check(lib().qk_apply_gate_full(self.ptr, iptr(words), len(words), dptr(params), nparams))

    def sqs(self, part, out_set, in_set, cl, start, stop):
        a = np.ascontiguousarray(out_set, dtype=np.int32)
        b = np.ascontiguousarray(in_set, dtype=np.int32)
        check(lib().qk_sqs(self.ptr, part, iptr(a), iptr(b), len(a), cl, start, stop))

    def csqs(self, local_set, rank_set):
        a = np.ascontiguousarray(local_set, dtype=np.int32)
        b = np.ascontiguousarray(rank_set, dtype=np.int32)
        check(lib().qk_csqs(self.ptr, iptr(a), iptr(b), len(a)))

    def sync(self):
        check(lib().qk_sync(self.ptr))

    def mark(self, slot: int):
        check(lib().qk_mark(self.ptr, slot))

    def mark_elapsed_ms(self, a: int, b: int) -> float:
        v = c_dbl(0.0)
        check(lib().qk_mark_elapsed(self.ptr, a, b, ctypes.byref(v)))
        return v.value
