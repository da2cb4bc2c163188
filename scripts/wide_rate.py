"""Zinc COEFF (and vanilla NTT) ct/s on the paper-parameter workloads (f3) from slots.
python scripts/wide_rate.py   (development tool)"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

out = {}
for name in ("P_bitcoin", "P_hg38"):
    cfg = CONFIGS[name]
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    _, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
    B = min(cfg.batch, 4096)
    zd = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
    m = Z.ckks_encode_batch_wide(ctx, zd)
    ct = ctx.empty_ct(B)
    r = {}
    for pname, fn in (("slots", lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, 1, 0, out=ct)),
                      ("i128", lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, m, 1, 0, out=ct))):
        fn()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        byt = B * (2 * cfg.L * cfg.n * 8 + (cfg.n // 2 * 8 if pname == "slots" else cfg.n * 16))
        r[pname] = {"ct_per_s": B / ms * 1e3, "hbm_frac": byt / (ms / 1e3) / 1e9 / 6549.1}
    Z.profile_enable(True)
    Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, 1, 0, out=ct)
    torch.cuda.synchronize()
    r["kernels"] = Z.profile_read()
    Z.profile_enable(False)
    out[name] = r
    del ct, zd, m
    ctx.close()
print(json.dumps(out))
