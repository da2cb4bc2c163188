"""Zinc COEFF from 128-bit plaintexts at P_hg38 (f3), a few calls (ncu target):
python scripts/run_wide_once.py [batch]  (development tool)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

cfg = CONFIGS["P_hg38"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
_, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
zd = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
m = Z.ckks_encode_batch_wide(ctx, zd)
ct = ctx.empty_ct(B)
for _ in range(3):
    Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, m, 1, 0, out=ct)
torch.cuda.synchronize()
print("ok")
