"""Split (S-CTA cluster) transform kernels vs the 2-CTA kernels on the same inputs:
reports mismatching (message, component, limb) and the index pattern.  Development tool.
python scripts/split_check.py [config] [batch] [scheme] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, int_plaintexts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
scheme = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = CONFIGS[name]
t = 65537 if scheme else 0
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale, scheme=scheme, t=t)
sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = {f: Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, f) for f in (Z.NTT, Z.COEFF)}
mm = int_plaintexts(cfg.log_n, B, seed=1, bound_bits=40)
m = torch.from_numpy(mm % t if t else mm).cuda()
calls = {"zinc_ntt": lambda: Z.zinc_encrypt_batch(ctx, cache[Z.NTT], Z.NTT, m, 7, 40),
         "vanilla_ntt": lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, m, 7, 40),
         "vanilla_coeff": lambda: Z.ckks_encrypt_batch(ctx, pk, Z.COEFF, m, 7, 40)}
bad = 0
for pname, fn in calls.items():
    Z.tune(Z.TUNE_SPLIT, 0)
    ref = fn().cpu().numpy()
    Z.tune(Z.TUNE_SPLIT, 1)
    for rep in range(reps):
        got = fn().cpu().numpy()
        diff = got != ref
        if diff.any():
            bad += 1
            idx = np.argwhere(diff)
            msgs = sorted(set(idx[:, 0].tolist()))
            print(f"{pname} rep {rep}: {diff.sum()} words differ in {len(msgs)} msgs {msgs[:10]}")
            for b in msgs[:3]:
                sub = idx[idx[:, 0] == b]
                comps = sorted(set(map(tuple, sub[:, 1:3].tolist())))
                pos = sub[:, 3]
                print(f"   msg {b}: (comp, limb) {comps[:8]} positions {pos.min()}..{pos.max()} count {len(pos)} "
                      f"mod8 {np.bincount(pos % 8, minlength=8).tolist()}")
    Z.tune(Z.TUNE_SPLIT, 1)
_, st, _ = Z.ckks_decrypt_batch(ctx, sk, Z.NTT, calls["zinc_ntt"](), slots=False)
print("decrypt status sum", int(st.sum()))
print("split_check", name, "scheme", scheme, "bad runs", bad)
