"""One small-batch call per path (ncu target for the latency path).
python scripts/small_once.py <batch> [knob SMALL_CLUSTER]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if len(sys.argv) > 2:
    Z.tune(Z.TUNE_SMALL_CLUSTER, int(sys.argv[2]))
cfg = CONFIGS["C5"]
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = {f: Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, f) for f in (Z.COEFF, Z.NTT)}
z = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
for _ in range(3):
    Z.zinc_encrypt_batch(ctx, cache[Z.COEFF], Z.COEFF, z, 1, 0)
    Z.ckks_encrypt_batch(ctx, pk, Z.NTT, z, 1, 0)
torch.cuda.synchronize()
