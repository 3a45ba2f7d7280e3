"""`Quokka` / `quokka sim` command line — mirror of the reference's simulation
entry point (/root/reference/pkg/src/quokka/cli.py:124-202, 307-335).

    python -m paper_2406_14084_b200 -i cfg.ini -c circuit.txt [--amps K] [--amps-file P]

Same .ini rules, same chunk-size inference from the circuit, same stdout
report and `error: ...` / exit status 1 behaviour. The optimized text is parsed
natively (qk_load_text) and simulated on the GPU. The other reference
subcommands (gen, finder, validate, bench) belong to the optimizer/harness and
stay with the reference package.
"""
from __future__ import annotations

import argparse
import configparser
import os
import sys
import time

from . import _lib
from .circuit import LayoutParams
from .errors import ParseError, SimulationError


class CliError(Exception):
    pass


def _workers() -> int:                                    # cli.py:40-44
    try:
        return max(1, int(os.environ.get("QUOKKA_WORKERS", "1")))
    except ValueError:
        return 1


def _read_text(path: str) -> str:                         # cli.py:47-52
    try:
        with open(path, "r", encoding="utf-8") as fh:
            return fh.read()
    except OSError as exc:
        raise CliError(f"cannot read {path}: {exc.strerror}")


def scan_optimized(text: str):
    """(max block gate target, min CSQS rank position) — cli.py:66-91."""
    max_target, min_rank = 0, None
    rows = [r for r in (ln.split("#", 1)[0].split() for ln in text.splitlines()) if r]
    i = 0
    two_q = ("CX", "CP", "SWAP", "RZZ")
    while i < len(rows):
        try:
            count = int(rows[i][0])
            for toks in rows[i + 1:i + 1 + count]:
                head = toks[0]
                if head == "CSQS":
                    m = int(toks[1])
                    ranks = [int(x) for x in toks[2 + m:2 + 2 * m]]
                    if ranks:
                        low = min(ranks)
                        min_rank = low if min_rank is None else min(min_rank, low)
                elif head != "SQS":
                    if head.startswith("D") and head[1:].isdigit():
                        arity = int(head[1:])
                    else:
                        arity = 2 if head in two_q else 1
                    for tok in toks[1:1 + arity]:
                        max_target = max(max_target, int(tok))
        except (ValueError, IndexError):
            raise CliError(f"bad optimized circuit structure near {' '.join(rows[i])!r}")
        i += 1 + count
    return max_target, min_rank


def load_ini(path: str) -> LayoutParams:                  # cli.py:124-151
    cp = configparser.ConfigParser(inline_comment_prefixes=("//", "#", ";"))
    try:
        with open(path, "r", encoding="utf-8") as fh:
            cp.read_file(fh, source=path)
    except OSError as exc:
        raise CliError(f"cannot read {path}: {exc.strerror}")
    except configparser.Error as exc:
        raise CliError(f"bad config {path}: {exc}")
    if cp.sections() != ["system"]:
        raise CliError(f"{path}: expected exactly one [system] section")
    keys = set(cp["system"])
    want = {"total_qbit", "rank_qbit", "buffer_qbit"}
    if keys != want:
        odd = sorted(keys - want) + sorted(want - keys)
        raise CliError(f"{path}: config keys must be exactly total_qbit, rank_qbit, "
                       f"buffer_qbit (offending: {', '.join(odd)})")
    try:
        n = cp.getint("system", "total_qbit")
        r = cp.getint("system", "rank_qbit")
        b = cp.getint("system", "buffer_qbit")
    except ValueError as exc:
        raise CliError(f"{path}: {exc}")
    if not (0 <= r <= n):
        raise CliError(f"{path}: need 0 <= rank_qbit <= total_qbit")
    if not (0 <= b <= n - r):
        raise CliError(f"{path}: need buffer_qbit <= total_qbit - rank_qbit")
    return LayoutParams(n=n, c=n - r, r=r, cl=min(2, n - r), b=b)


def cmd_sim(args) -> int:                                 # cli.py:154-202
    from .simulator import Simulator
    base = load_ini(args.config)
    text = _read_text(args.circuit)
    max_target, _ = scan_optimized(text)
    c = max_target + 1
    if c > base.local_qubits:
        raise CliError(
            f"circuit targets chunk qubit {max_target} but only {base.local_qubits} "
            f"local qubits are available with rank_qbit={base.r}")
    layout = LayoutParams(n=base.n, c=c, r=base.r, cl=min(2, c), b=base.b)
    _lib.parse_text(text, layout.n, layout.local_qubits, layout.c)   # parse errors before allocation
    workers = _workers()
    sim = Simulator(layout, workers_per_rank=workers)
    perm = sim.load_text(text, c)
    t0 = time.perf_counter()
    res = sim.run_loaded(perm)
    wall = time.perf_counter() - t0

    print(f"qubits {layout.n}  ranks {layout.num_ranks}  chunk_qubits {layout.c}  "
          f"cacheline_qubits {layout.cl}  buffer_qubits {layout.b}  workers {workers}")
    print(f"norm {res.norm():.12f}")
    print(f"elapsed_seconds {wall:.6f}")
    print(f"gate_seconds {res.timings['gate']:.6f}")
    print(f"ims_seconds {res.timings['ims']:.6f}")
    print(f"xrs_seconds {res.timings['xrs']:.6f}")
    print("aio_seconds 0.000000")

    k = args.amps
    if k or args.amps_file:
        k = min(k or (1 << layout.n), 1 << layout.n)
        vals = res.logical_amplitudes(k)
        pairs = [(float(v.real), float(v.imag)) for v in vals]
        if args.amps_file:
            with open(args.amps_file, "w", encoding="utf-8") as fh:
                for re_, im in pairs:
                    fh.write(f"{re_!r} {im!r}\n")
        else:
            for i, (re_, im) in enumerate(pairs):
                print(f"amp {i} {re_!r} {im!r}")
    return 0


def _add_sim_args(p: argparse.ArgumentParser) -> None:   # cli.py:254-260
    p.add_argument("-i", dest="config", required=True, help=".ini configure file")
    p.add_argument("-c", dest="circuit", required=True, help="optimized circuit file")
    p.add_argument("--amps", type=int, default=0, metavar="K",
                   help="print the first K logical amplitudes")
    p.add_argument("--amps-file", default=None, metavar="PATH",
                   help="write amplitudes (re im per line) to PATH instead of stdout")


def _run(func, args) -> int:                              # cli.py:307-312
    try:
        return func(args)
    except (CliError, ParseError, SimulationError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


def sim_main(argv=None) -> int:                           # cli.py:330-335
    parser = argparse.ArgumentParser(prog="Quokka", description="Simulate an optimized circuit.")
    _add_sim_args(parser)
    return _run(cmd_sim, parser.parse_args(argv))


def main(argv=None) -> int:
    """`quokka sim ...` subcommand form (cli.py:271-273)."""
    parser = argparse.ArgumentParser(prog="quokka")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("sim", help="simulate an optimized circuit")
    _add_sim_args(p)
    p.set_defaults(func=cmd_sim)
    args = parser.parse_args(argv)
    return _run(args.func, args)


if __name__ == "__main__":
    sys.exit(sim_main())
