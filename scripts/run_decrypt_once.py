"""Runs the batched COEFF-form decrypt + decode a few times (for ncu):
python scripts/run_decrypt_once.py [config] [batch]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, int_plaintexts  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
m = torch.from_numpy(int_plaintexts(cfg.log_n, 64, seed=1, bound_bits=40)).cuda().repeat(B // 64, 1)
ct = Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, m, 1, 0)
for _ in range(3):
    Z.ckks_decrypt_batch(ctx, sk, Z.COEFF, ct)
torch.cuda.synchronize()
print("ok")
