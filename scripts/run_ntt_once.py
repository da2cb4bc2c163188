"""Runs one NTT-bound path a few times (for ncu): python scripts/run_ntt_once.py
{zinc_ntt|vanilla_ntt|vanilla_coeff|decrypt|int_peak<V>} [config] [batch]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, int_plaintexts  # noqa: E402

which = sys.argv[1]
if os.environ.get("ZINC_SPLIT") is not None:
    Z.tune(Z.TUNE_SPLIT, int(os.environ["ZINC_SPLIT"]))
cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C3"]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
_, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.NTT)
m = torch.from_numpy(int_plaintexts(cfg.log_n, 64, seed=1, bound_bits=44)).cuda().repeat(B // 64, 1)
ct = ctx.empty_ct(B)
for _ in range(3):
    if which.startswith("int_peak"):
        Z.zinc_int_peak(ctx, 148 * 8, 500, torch.zeros(2, dtype=torch.uint64, device="cuda"), variant=int(which[-1]))
    elif which == "decrypt":
        Z.ckks_decrypt_batch(ctx, Z.zinc_keygen(ctx, cfg.key_seed)[0], Z.COEFF, ct, slots=False)
    elif which == "zinc_ntt":
        Z.zinc_encrypt_batch(ctx, cache, Z.NTT, m, 1, 0, out=ct)
    elif which == "vanilla_ntt":
        Z.ckks_encrypt_batch(ctx, pk, Z.NTT, m, 1, 0, out=ct)
    else:
        Z.ckks_encrypt_batch(ctx, pk, Z.COEFF, m, 1, 0, out=ct)
torch.cuda.synchronize()
print("ok")
