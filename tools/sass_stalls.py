"""Summarise an ncu source page (SASS, csv, gzipped): stall samples and
instruction counts by opcode, plus the hottest instructions.

    python tools/sass_stalls.py gpurun_out/r02z/p6_source_sass.csv.gz
"""
import collections
import csv
import gzip
import io
import re
import sys

rows = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
hdr, data = rows[1], rows[2:]
ix = {k: i for i, k in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError):
        return 0.0


by, inst = collections.Counter(), collections.Counter()
stall = collections.defaultdict(collections.Counter)
skeys = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
for r in data:
    src = r[ix["Source"]].strip()
    op = re.sub(r"^@!?U?P\d+\s+", "", src).split()[0].split(".")[0] if src else "?"
    by[op] += f(r, "Warp Stall Sampling (All Samples)")
    inst[op] += f(r, "Instructions Executed")
    for k in skeys:
        stall[op][k] += f(r, k)
tot, ti = sum(by.values()), sum(inst.values())
print(f"samples {int(tot)}  warp instructions {int(ti)}  smem wavefronts {int(sum(f(r, 'L1 Wavefronts Shared') for r in data))}"
      f" (ideal {int(sum(f(r, 'L1 Wavefronts Shared Ideal') for r in data))})")
for op, v in by.most_common(16):
    top = ", ".join(f"{k[6:]}={int(c)}" for k, c in stall[op].most_common(3))
    print(f"{op:10s} samples {100 * v / tot:5.1f}%  inst {100 * inst[op] / ti:5.1f}%  {top}")
print("hottest:")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:12]:
    print(f"  {r[ix['Source']].strip()[:64]:64s} {int(f(r, 'Warp Stall Sampling (All Samples)'))}")
