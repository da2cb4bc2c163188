"""Per-butterfly SASS mix of the K11 variants (int_peak_kernel<V>, k_stream.cu): the
opcodes of the main loop (between its backward branch and the branch target; one trip =
8 butterflies), less the loop's own counter / branch instructions, divided by 8.
fma pipe = the IMAD family plus HFMA2 (B300_MICROARCH.md: FFMA/FMUL/IMAD/HFMA2).
Usage: python scripts/sass_bfly.py [k_stream.o]  (run after build; no GPU needed)"""
import collections
import re
import subprocess
import sys

obj = sys.argv[1] if len(sys.argv) > 1 else "paper_2408_07304_b200/build/k_stream.o"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
NAMES = {0: "ct_bfly", 1: "ct_bfly_nr", 2: "ct_bfly_a", 3: "gs_bfly"}
LOOP_OVERHEAD = ("UIADD3", "UISETP", "BRA", "UMOV", "LOP3")  # counter, exit test, branch, w += v[0] & 1
res = {}
for f in re.split(r"\n\s*Function : ", sass)[1:]:
    m = re.match(r"_ZN4zinc15int_peak_kernelILi(\d)E", f.split("\n", 1)[0].strip())
    if not m:
        continue
    ins = [(int(a, 16), t.strip()) for a, t in re.findall(r"/\*([0-9a-f]{4})\*/\s+([^;]*);", f)]
    loop = None
    for a, t in ins:
        b = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", t)
        if b and int(b.group(1), 16) < a and (loop is None or a - int(b.group(1), 16) > loop[1] - loop[0]):
            loop = (int(b.group(1), 16), a)
    ops = collections.Counter()
    for a, t in ins:
        if loop[0] <= a <= loop[1]:
            w = t.split()
            ops[w[1] if w[0].startswith("@") else w[0]] += 1
    body = {k: v for k, v in ops.items() if not k.startswith(LOOP_OVERHEAD)}
    n = sum(body.values())
    fma = sum(v for k, v in body.items() if k.startswith(("IMAD", "HFMA2", "FFMA", "FMUL")))
    # butterflies per loop trip: 8 per source iteration times ptxas's unroll factor; the
    # 3-partial-product Shoup quotient (variants 1-3) has exactly two IMAD.HI.U32 per butterfly
    v = int(m.group(1))
    nb = 8 if v == 0 else max(8, 8 * round(body.get("IMAD.HI.U32", 16) / 16))
    res[v] = (n / nb, fma / nb, body)
for v in sorted(res):
    n, fma, body = res[v]
    print(f"{v} {NAMES[v]:11s} instr/bfly {n:6.3f}  fma-pipe/bfly {fma:6.3f}  other/bfly {n - fma:6.3f}  "
          f"{dict(sorted(body.items()))}")
