"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
gate-block passes of one tuned QAOA30 run, from the `ncu --set full` capture of
tools/r02v.sh (raw page, gzipped csv) -> profiles/traffic.json. Measured on the
headline configuration itself, no scaling.

    python tools/traffic.py gpurun_out/r02v/full_qaoa30/raw.csv.gz r02v
"""
import csv
import gzip
import io
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, tag):
    rows = list(csv.reader(io.StringIO(gzip.open(path, "rt").read())))
    hdr, units = rows[0], rows[1]
    per = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))

        def val(k):
            return float(d[k].replace(",", "")) * UNITS.get(units[hdr.index(k)], 1)

        per.append({"kernel": d["Kernel Name"], "ms": float(d["gpu__time_duration.sum"].replace(",", "")),
                    "dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum")})
    avg = sum(p["dram_read"] + p["dram_write"] for p in per) / len(per)
    out = {"_how": f"ncu --set full of the {len(per)} gate-block passes of one tuned qaoa30 run "
                   f"(tools/r02v.sh, capture {tag}); k_block_tma = mean dram__bytes_read.sum + "
                   "dram__bytes_write.sum per launch. The first passes after qk_reset read only "
                   "the zero-support prefix (bounded TMA view), so their traffic is mostly writes.",
           "qaoa30": {"k_block_tma": avg, "launches": per}}
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print(f"{len(per)} launches, mean {avg / 1e9:.2f} GB per launch")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
