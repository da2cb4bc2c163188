"""One-screen comparison of ncu raw CSV captures (ncu --page raw --csv):
python scripts/ncu_brief.py gpurun_out/<tag>/raw_<name>.csv ..."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "dur"), ("sm__inst_executed.sum", "inst"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_inst%"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_inst%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankconf"),
        ("launch__registers_per_thread", "regs"), ("launch__occupancy_limit_registers", "lim_reg"),
        ("launch__occupancy_limit_shared_mem", "lim_smem"), ("launch__grid_size", "grid")]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    out = []
    for k, n in KEYS:
        if k in d:
            out.append(f"{n}={d[k]}")
    stalls = {h.split("smsp__average_warp_latency_issue_stalled_")[1].split(".")[0]: float(v)
              for h, v in d.items() if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")
              and v not in ("", "n/a")}
    if not stalls:
        stalls = {h.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(v.replace(",", ""))
                  for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and v not in ("", "n/a")
                  and not h.endswith("_not_issued")}
    top = sorted(stalls.items(), key=lambda x: -x[1])[:8]
    print(path.split("/")[-1], d.get("Kernel Name", "")[:60])
    print("  " + " ".join(out))
    print("  stalls: " + " ".join(f"{k}={v:.3g}" for k, v in top))
