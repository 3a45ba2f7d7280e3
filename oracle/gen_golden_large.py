"""Full-size golden samples FROM THE REFERENCE ITSELF (test infrastructure).

Run in the build container (where /root/reference is importable, 62 GB RAM):

    python oracle/gen_golden_large.py qaoa30_c12_r0 [workers]

It parses `bench_circuits/<name>.txt` with the reference parser, runs the
reference `Simulator(layout, workers_per_rank=workers).run(opt)` (simulator.py:529-555)
on the full 2^n state, and stores into `tests/golden/large_<name>.npz`:

  idx      65,536 sorted random physical indices (seed 11) plus 0 and 2^n-1
  amps     the reference's physical amplitudes at those indices
  norm     SimResult.norm() (simulator.py:393-397)
  perm     the final permutation (circuit.py:202-210)
  timings  the reference's per-class seconds and the wall time, with the
           core count: a measured (not extrapolated) CPU reference time

Nothing on the GPU box reads /root/reference; the -m gpu test
`test_reference_full_size_qaoa30` only reads the committed npz.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("QUOKKA_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from quokka.circuit import LayoutParams, parse_optimized  # noqa: E402
from quokka.simulator import Simulator  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "qaoa30_c12_r0"
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
    fam = name.split("_")
    n = int("".join(ch for ch in fam[0] if ch.isdigit()))
    c = int(fam[1][1:])
    r = int(fam[2][1:])
    with open(os.path.join(ROOT, "bench_circuits", name + ".txt")) as fh:
        text = fh.read()
    lay = LayoutParams(n=n, c=c, r=r)
    opt = parse_optimized(text, lay)
    t0 = time.perf_counter()
    sim = Simulator(lay, workers_per_rank=workers)
    t1 = time.perf_counter()
    res = sim.run(opt)
    t2 = time.perf_counter()
    sim.close()
    norm = res.norm()
    t3 = time.perf_counter()
    rng = np.random.default_rng(11)
    size = 1 << n
    idx = np.unique(np.concatenate([rng.integers(0, size, 65536, dtype=np.int64),
                                    np.array([0, size - 1], dtype=np.int64)]))
    local = 1 << lay.local_qubits
    amps = np.empty(idx.size, dtype=np.complex128)
    for k, p in enumerate(res.partitions):
        sel = (idx >> lay.local_qubits) == k
        amps[sel] = p.amps[idx[sel] & (local - 1)]
    info = {"name": name, "n": n, "c": c, "r": r, "workers": workers,
            "cpu_count": os.cpu_count(), "init_s": t1 - t0, "run_s": t2 - t1,
            "norm_s": t3 - t2, "timings": res.timings,
            "instructions": len(opt.instructions)}
    out = os.path.join(ROOT, "tests", "golden", f"large_{name}.npz")
    np.savez_compressed(out, idx=idx, amps=amps, norm=np.float64(norm),
                        perm=np.asarray(res.final_permutation, dtype=np.int64),
                        info=np.array(json.dumps(info)))
    print(json.dumps(info))


if __name__ == "__main__":
    main()
