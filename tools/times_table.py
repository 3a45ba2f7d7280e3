"""Summarise a pass_times log: one line per configuration with per-pass ms."""
import re
import sys

cur, out = None, {}
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line.strip()
        out[cur] = []
        continue
    m = re.search(r"instr (\d+).*: ([\d.]+) ms", line)
    if m:
        out[cur].append(float(m.group(2)))
    elif cur and line.strip():
        out[cur].append(line.strip()[:160])
for k, v in out.items():
    nums = [x for x in v if isinstance(x, float)]
    errs = [x for x in v if not isinstance(x, float)]
    print(f"{k:45s} n={len(nums):3d} sum={sum(nums):7.2f}", " ".join(f"{x:.2f}" for x in nums[:16]), errs[-1:] if errs else "")
