"""Runs the persistent pipeline a few times (for ncu): C3, knobs from argv
(enc, mpc, variant, ring)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

enc, mpc, variant, ring = [int(x) for x in (sys.argv[1:] + ["92", "8", "0", "256"][len(sys.argv) - 1:])]
cfg = CONFIGS["C3"]
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
_, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
slots = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, cfg.batch))).cuda()
ct = ctx.empty_ct(cfg.batch)
for k, v in {Z.TUNE_OVERLAP: 3, Z.TUNE_PIPE_ENC_CTAS: enc, Z.TUNE_COEFF_MSGS_PER_CTA: mpc,
             Z.TUNE_PIPE_VARIANT: variant, Z.TUNE_ENCODE_CHUNK_BYTES: ring * cfg.n * 8}.items():
    Z.tune(k, v)
for _ in range(3):
    Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, slots, 1, 0, out=ct)
torch.cuda.synchronize()
print("ok")
