"""Refresh profiles/ncu_traffic.json (the `traffic` of bench.py's roofline) from one
gpu_round.sh session: dram__bytes_read.sum + dram__bytes_write.sum of each captured
kernel's single `ncu --set full` launch (one launch of the bench's C3 run), per message; the
messages of the launch follow from its grid (CTAs per message below).
Usage: python scripts/update_traffic.py <tag>"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# CTAs per message of each captured kernel at C3 (N = 2^14, L = 8): the Zinc COEFF kernel runs
# 32 coefficient tiles x (messages / 2) groups; the cluster kernels 4 CTAs, the 2-CTA kernels 2,
# the complex encode (C4's, N = 2^15: the only complex-slot encode the bench runs) 2, the real
# encode 1.
CTAS_PER_MSG = {"zinc_coeff_kernel": 16, "zinc_ntt_split": 4, "vanilla_coeff_split": 4, "decrypt_split": 4,
                "vanilla_ntt_dit": 2, "encode_kernel": 2, "encode_real_kernel": 1}


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
        msgs = max(1, round(grid / CTAS_PER_MSG.get(kernel, 1)))
        out[kernel] = {"config": "C4" if kernel == "encode_kernel" else "C3", "msgs_per_launch": msgs, "dram_bytes_per_msg": round(tot / msgs),
                       "grid": grid,
                       "source": f"gpurun_out/{tag} (ncu --set full of one launch of the bench's C3 run, "
                                 f"{msgs} messages; ncu flushes caches)"}
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
