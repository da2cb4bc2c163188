"""Refresh profiles/ncu_traffic.json (the `traffic` of bench.py's roofline) from one
gpu_round.sh session: dram__bytes_read.sum + dram__bytes_write.sum of each captured
kernel's single `ncu --set full` launch (the bench's C3 chunk of 256 messages), per
message.  Usage: python scripts/update_traffic.py <tag>"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    tag = sys.argv[1]
    src = os.path.join(ROOT, "gpurun_out", tag)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for f in sorted(os.listdir(src)):
        if not (f.startswith("raw_") and f.endswith(".csv")):
            continue
        kernel = f[4:-4]
        rows = list(csv.reader(open(os.path.join(src, f))))
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u, v = d[k]
            tot += float(v.replace(",", "")) * SCALE.get(u, 1)
        grid = float(d.get("launch__grid_size", ("", "0"))[1].replace(",", "") or 0)
        msgs = 256
        out[kernel] = {"config": "C3", "msgs_per_launch": msgs, "dram_bytes_per_msg": round(tot / msgs),
                       "grid": grid,
                       "source": f"gpurun_out/{tag} (profiles/r01_ncu_summary.*: ncu --set full, one launch of the "
                                 "bench's C3 chunk of 256 messages; ncu flushes caches)"}
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
