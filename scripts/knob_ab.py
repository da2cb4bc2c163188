"""A/B of one tuning knob on the Zinc COEFF-from-slots step at C2 / C3 / C4, alternating the
values, median of 5 per measurement: python scripts/knob_ab.py <knob> <v0> <v1> [configs]
(development tool)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


knob, vals = int(sys.argv[1]), [int(sys.argv[2]), int(sys.argv[3])]
names = (sys.argv[4] if len(sys.argv) > 4 else "C2,C3,C4").split(",")
for name in names:
    cfg = CONFIGS[name]
    B = {"C2": 4096, "C3": 16384, "C4": 4096}[name]
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    _, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
    z = slots_batch(cfg, 0, B)
    if cfg.complex_slots:
        z = np.stack([z.real, z.imag], axis=-1)
    zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    ct = ctx.empty_ct(B)
    byt = B * (2 * cfg.L * cfg.n * 8 + cfg.n * 8)
    res = {v: [] for v in vals}
    for rep in range(int(os.environ.get("AB_REPS", "3"))):
        for v in (vals if rep % 2 == 0 else vals[::-1]):
            old = Z.tune(knob, v)
            time.sleep(float(os.environ.get("AB_COOL_S", "3")))  # sustained HBM load slows the GPU: start cool
            res[v].append(round(timeit(lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, 3, 0, out=ct)), 4))
            Z.tune(knob, old)
    print(name, json.dumps({v: {"ms": r, "hbm_frac": [round(byt / (x * 1e-3) / 1e9 / 6547.2, 4) for x in r]}
                            for v, r in res.items()}), flush=True)
    del ct, zd
    torch.cuda.empty_cache()
