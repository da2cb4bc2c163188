"""Stall reasons by region (regions cut at barrier-like instructions, as ncu_regions.py) and the
top instructions for one stall reason: python scripts/ncu_stall_regions.py source.csv.gz [reason] [top]"""
import collections
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
CUT = ("BAR.SYNC", "SYNCS.PHASECHK", "UCGABAR_WAIT", "SYNCS.ARRIVE")
REASONS = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
num = lambda r, k: float(r[ci[k]] or 0)
tot = {k: sum(num(r, k) for r in body) for k in REASONS}
T = sum(tot.values())
print("overall:", ", ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
reg = collections.Counter()
start = 0
for idx, r in enumerate(body):
    for k in REASONS:
        reg[k] += num(r, k)
    src = r[ci["Source"]].strip()
    if any(src.startswith(c) or (" " + c) in src for c in CUT) or idx == len(body) - 1:
        s = sum(reg.values())
        if s > 0.01 * T:
            print(f"[{start:5d}-{idx:5d}] {100 * s / T:5.1f}%  " +
                  ", ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in sorted(reg.items(), key=lambda x: -x[1])[:5]) + f"  | {src[:30]}")
        reg = collections.Counter()
        start = idx + 1
print(f"top {reason}:")
for idx, r in sorted(enumerate(body), key=lambda x: -num(x[1], reason))[:top]:
    print(f"  {idx:5d} {100 * num(r, reason) / T:5.2f}%  {r[ci['Source']].strip()[:70]}")
