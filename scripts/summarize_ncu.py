"""Summarise one gpu_round.sh session (gpurun_out/<tag>/) into profiles/:
per-kernel `ncu --set full` metrics (duration, DRAM bytes, throughput, issue /
pipe utilisation, top stall reasons, registers, shared memory), the launch
list's per-kernel shares, and the bench line.  Usage:
    python scripts/summarize_ncu.py <tag> [out-prefix]"""
import csv
import gzip
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "pipe_alu_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "pipe_fma_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "pipe_fp64_pct"),
    ("sm__inst_executed.sum", "inst_executed"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "smem_dynamic"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
]


US = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def to_bytes(v, unit):
    x = float(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return x * scale.get(unit, 1)


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name")}
    for m, name in METRICS:
        if m in d and d[m] not in ("", "n/a"):
            v = d[m].replace(",", "")
            try:
                if "bytes" in m:
                    out[name] = to_bytes(v, u[m])
                elif m == "gpu__time_duration.sum":
                    out[name + "_us"] = float(v) * US[u[m]]
                else:
                    out[name] = float(v)
            except ValueError:
                out[name] = v
    st = [(h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v))
          for h, v in d.items() if h.startswith("smsp__average_warps_issue_stalled_")
          and h.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
    out["top_stalls_per_issue"] = dict(sorted(st, key=lambda x: -x[1])[:6])
    return out


def launch_shares(path):
    if path.endswith(".gz"):
        f = gzip.open(path, "rt")
    else:
        f = open(path)
    lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    I = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[I["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[I["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0].replace("zinc::", "")
        v = float(r[I["Metric Value"]].replace(",", ""))
        unit = r[I["Metric Unit"]]
        us = v * US[unit]
        tot[name] += us
        cnt[name] += 1
    s = sum(tot.values())
    return {k: {"launches": cnt[k], "total_us": tot[k], "share": tot[k] / s} for k in sorted(tot, key=lambda k: -tot[k])}


def main():
    tag = sys.argv[1]
    prefix = sys.argv[2] if len(sys.argv) > 2 else tag
    src = os.path.join(ROOT, "gpurun_out", tag)
    out = {"session": tag, "kernels": {}}
    for f in sorted(os.listdir(src)):
        if f.startswith("raw_") and f.endswith(".csv"):
            out["kernels"][f[4:-4]] = raw_metrics(os.path.join(src, f))
    for name in ("launches.csv.gz", "launches.csv"):
        if os.path.exists(os.path.join(src, name)):
            out["launch_list_shares"] = launch_shares(os.path.join(src, name))
            break
    if os.path.exists(os.path.join(src, "bench.json")):
        try:
            out["bench"] = json.loads(open(os.path.join(src, "bench.json")).read().strip().splitlines()[-1])
        except (ValueError, IndexError):
            pass
    dst = os.path.join(ROOT, "profiles", f"{prefix}_ncu_summary.json")
    json.dump(out, open(dst, "w"), indent=1)
    lines = [f"# ncu summary: {tag}", ""]
    for k, m in out["kernels"].items():
        lines.append(f"## {k}")
        for kk, vv in m.items():
            lines.append(f"- {kk}: {vv}")
        lines.append("")
    if "launch_list_shares" in out:
        lines.append("## launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)")
        for k, v in out["launch_list_shares"].items():
            lines.append(f"- {k}: {v['launches']} launches, {v['total_us']:.1f} us, share {v['share']:.3f}")
    open(os.path.join(ROOT, "profiles", f"{prefix}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    print(dst)


if __name__ == "__main__":
    main()
