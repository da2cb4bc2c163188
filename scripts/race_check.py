"""Repeatability stress: the bench's Zinc COEFF call from slots at C3 (B messages), encrypted
twice (bitwise equal?) and decrypted repeatedly in COEFF form with both transform-kernel
families (CRT status all zero?).  python scripts/race_check.py [B] [reps]  (development tool)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = CONFIGS["C3"]
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = {f: Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, f) for f in (Z.COEFF, Z.NTT)}
zd = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
res = {}
for path, form in (("zinc", Z.COEFF), ("zinc", Z.NTT), ("vanilla", Z.COEFF), ("vanilla", Z.NTT)):
    enc = (lambda: Z.zinc_encrypt_batch(ctx, cache[form], form, zd, 5, 0)) if path == "zinc" else \
          (lambda: Z.ckks_encrypt_batch(ctx, pk, form, zd, 5, 0))
    ref = enc()
    diff_enc = 0
    for _ in range(3):
        diff_enc += int((enc() != ref).any(dim=(1, 2, 3)).sum())
    bad = {}
    for split in (1, 0):
        Z.tune(Z.TUNE_SPLIT, split)
        n = 0
        for _ in range(reps):
            _, st, _ = Z.ckks_decrypt_batch(ctx, sk, form, ref, slots=False)
            n += int(st.sum())
        bad[split] = n
    Z.tune(Z.TUNE_SPLIT, 1)
    res[f"{path}_{'coeff' if form else 'ntt'}"] = {"enc_msgs_differing": diff_enc, "dec_bad_split1": bad[1],
                                                    "dec_bad_split0": bad[0]}
    print(res, flush=True)
