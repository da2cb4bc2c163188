"""Instruction mix of an ncu source-page export (SASS view) by region: the kernel is cut
at every barrier-like instruction (BAR, SYNCS, UCGABAR, MEMBAR) and each region reports
its executed warp-instructions by class, its stall samples, and per-butterfly figures.
python scripts/ncu_regions.py source_<name>.csv.gz [butterflies]"""
import collections
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
bfly = float(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
CUT = ("BAR.SYNC", "SYNCS.PHASECHK", "UCGABAR_WAIT", "SYNCS.ARRIVE")


def cls(op):
    if op.startswith(("IMAD", "HFMA2", "IMUL")):
        return "fma"
    if op.startswith(("LDS", "STS", "LDG", "STG", "LD.", "ST.", "LDL", "STL", "LDGSTS", "LD", "ST")):
        return "mem"
    if op.startswith(("BRA", "BSSY", "BSYNC", "EXIT", "RET", "CALL", "WARPSYNC")):
        return "ctl"
    return "alu"


regions = []
cur = collections.Counter()
samp = 0
start = 0
for idx, r in enumerate(body):
    src = r[ci["Source"]].strip()
    w = src.split()
    if not w:
        continue
    op = w[1] if w[0].startswith("@") else w[0]
    n = int(r[ci["Instructions Executed"]] or 0)
    cur[cls(op)] += n
    cur["all"] += n
    if op.startswith(("IMAD.MOV", "MOV", "HFMA2")):
        cur["moves"] += n
    samp += int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    if any(src.startswith(c) or (" " + c) in src for c in CUT):
        regions.append((start, idx, cur, samp, src[:40]))
        cur = collections.Counter()
        samp = 0
        start = idx + 1
regions.append((start, len(body) - 1, cur, samp, "end"))
tot = sum(r[2]["all"] for r in regions)
tots = sum(r[3] for r in regions)
print(f"total warp-instr {tot}  samples {tots}" + (f"  thread-instr/bfly {32 * tot / bfly:.2f}" if bfly else ""))
for a, b, c, s, tag in regions:
    if c["all"] < 0.002 * tot and s < 0.002 * tots:
        continue
    per = (lambda k: f"{32 * c[k] / bfly:5.2f}") if bfly else (lambda k: f"{c[k]:9d}")
    print(f"[{a:5d}-{b:5d}] instr {100 * c['all'] / tot:5.1f}%  samples {100 * s / tots:5.1f}%  "
          f"all {per('all')} fma {per('fma')} alu {per('alu')} mem {per('mem')} ctl {per('ctl')} moves {per('moves')}  | {tag}")
