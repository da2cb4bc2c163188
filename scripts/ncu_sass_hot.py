"""Stall samples of an ncu source-page export (SASS view) by opcode and the hottest
instructions: python scripts/ncu_sass_hot.py gpurun_out/<tag>/source_<name>.csv.gz [top]"""
import collections
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
inst = sum(int(r[ci["Instructions Executed"]] or 0) for r in body)
byop = collections.Counter()
byop_i = collections.Counter()
for r in body:
    src = r[ci["Source"]].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    op = op.split(".")[0]
    byop[op] += int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    byop_i[op] += int(r[ci["Instructions Executed"]] or 0)
print(f"samples {tot}  warp-instructions {inst}")
print("by opcode (share of samples / share of instructions):")
for op, v in byop.most_common(20):
    print(f"  {op:10s} {100 * v / tot:5.1f}%  {100 * byop_i[op] / inst:5.1f}%")
print("hottest instructions:")
for idx, r in sorted(enumerate(body), key=lambda x: -int(x[1][ci["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
    print(f"  {idx:5d} {int(r[ci['Warp Stall Sampling (All Samples)']]):6d} {r[ci['Source']].strip()[:90]}")
