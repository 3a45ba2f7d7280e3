"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
block, cluster-exchange and SQS passes from the qaoa26 `ncu --set full`
captures of tools/evidence.sh, scaled to one qaoa30 launch -> profiles/traffic.json.

    python tools/traffic.py gpurun_out/<tag> profiles/<tag>_ncu_full_qaoa26.txt
"""
import csv
import io
import json
import os
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))

        def val(k):
            return float(d[k].replace(",", "")) * UNITS.get(units[hdr.index(k)], 1)

        out.append((d["Kernel Name"], val("dram__bytes_read.sum") + val("dram__bytes_write.sum")))
    return out


def main(run_dir, summary):
    blk = launches(os.path.join(run_dir, "full_qaoa26.ncu-rep"))
    sqs = launches(os.path.join(run_dir, "full_sqs_qaoa26.ncu-rep"))
    jit = [b for k, b in blk if k.startswith("qk_jit") and not k.startswith("qk_jitx")]
    jx = [b for k, b in blk if k.startswith("qk_jitx")]
    sq = [b for _, b in sqs]
    alg = 32 * 2 ** 26
    t = {"_how": f"dram__bytes_read.sum + dram__bytes_write.sum per launch from {summary} (qaoa26: "
                 "2^26 amplitudes, 1 GiB state >> L2), divided by the launch's algorithmic bytes "
                 "(32 B x 2^26) and scaled to one qaoa30 launch (32 B x 2^30 = 34.36 GB). Dirty L2 "
                 "lines still resident at kernel end drain after it, hence write < read. Every "
                 "captured launch read a full state (none was the first pass after qk_reset).",
         "qaoa26": {"k_block_tma": sum(jit) / len(jit), "k_sqs": sum(sq) / len(sq),
                    "k_block_x": sum(jx) / max(1, len(jx)), "algorithmic_bytes": alg,
                    "launches": {"qk_jit": len(jit), "qk_jitx": len(jx), "k_sqs": len(sq)}}}
    t["qaoa30"] = {k: t["qaoa26"][k] * 16 for k in ("k_block_tma", "k_sqs", "k_block_x", "algorithmic_bytes")}
    with open("profiles/traffic.json", "w") as fh:
        json.dump(t, fh, indent=1)
    print(json.dumps(t["qaoa30"]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
