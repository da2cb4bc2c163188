"""Small-batch latency breakdown (C5): total device time of one call (CUDA events around it)
and the library's per-kernel traced times, for Zinc COEFF and vanilla NTT form at batch
1 and 16.  Development tool.  python scripts/latency.py [batches]"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

cfg = CONFIGS["C5"]
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = {f: Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, f) for f in (Z.COEFF, Z.NTT)}
out = {}
if os.environ.get("ZINC_SMALL_ENCODE") is not None:
    Z.tune(Z.TUNE_SMALL_ENCODE, int(os.environ["ZINC_SMALL_ENCODE"]))
if os.environ.get("ZINC_SMALL_CLUSTER") is not None:
    Z.tune(Z.TUNE_SMALL_CLUSTER, int(os.environ["ZINC_SMALL_CLUSTER"]))
for B in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,16").split(",")]:
    z = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
    ct = ctx.empty_ct(B)
    calls = {"zinc_coeff": lambda: Z.zinc_encrypt_batch(ctx, cache[Z.COEFF], Z.COEFF, z, 1, 0, out=ct),
             "zinc_ntt": lambda: Z.zinc_encrypt_batch(ctx, cache[Z.NTT], Z.NTT, z, 1, 0, out=ct),
             "vanilla_ntt": lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, z, 1, 0, out=ct),
             "encode": lambda: Z.ckks_encode_batch(ctx, z)}
    for name, fn in calls.items():
        for _ in range(3):
            fn()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        Z.profile_enable(True)
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        prof = {k: round(v[0] / v[1] * 1e3, 2) for k, v in Z.profile_read().items()}
        Z.profile_enable(False)
        out[f"{name}@{B}"] = {"us_median": round(statistics.median(ts), 2), "us_min": round(min(ts), 2),
                              "kernel_us": prof}
print(json.dumps(out, indent=1))
