"""C4 Zinc COEFF from complex slots (4096 messages): step time and HBM fraction, median of 5
(development tool; alternate libraries with ZINC_LIB_PATH for A/B)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

cfg = CONFIGS["C4"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
_, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
z = slots_batch(cfg, 0, B)
zd = torch.from_numpy(np.ascontiguousarray(np.stack([z.real, z.imag], axis=-1))).cuda()
ct = ctx.empty_ct(B)
ts = []
for it in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, 3, 0, out=ct)
    b.record()
    torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
enc = []
for it in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    Z.ckks_encode_batch(ctx, zd)
    b.record()
    torch.cuda.synchronize()
    enc.append(a.elapsed_time(b))
print(json.dumps({"ms": ms, "ct_per_s": B / ms * 1e3, "hbm_frac": B * (2 * cfg.L * cfg.n * 8 + cfg.n * 8) / (ms * 1e-3) / 1e9 / 6547.2,
                  "encode_ms": float(np.median(enc))}))
