"""Zinc COEFF-from-slots step time at C2, C3 and C4 (the bench's batches; C4 at 4096 messages),
CUDA events, median of 5, with the step's HBM fraction (ciphertext writes + int64 plaintext
bytes / measured copy bandwidth).  python scripts/zinc_coeff_steps.py  (development tool)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

peak = 6547.2
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


out = {}
for name, B in (("C2", 4096), ("C3", 16384), ("C4", 4096)):
    cfg = CONFIGS[name]
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    _, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
    z = slots_batch(cfg, 0, B)
    if cfg.complex_slots:
        z = np.stack([z.real, z.imag], axis=-1)
    zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    ct = ctx.empty_ct(B)
    ms = timeit(lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, 3, 0, out=ct))
    gbs = B * (2 * cfg.L * cfg.n * 8 + cfg.n * 8) / (ms * 1e-3) / 1e9
    out[name] = {"ms": round(ms, 4), "ct_per_s": round(B / ms * 1e3), "hbm_frac": round(gbs / peak, 4)}
    del ct, zd
    torch.cuda.empty_cache()
print(json.dumps(out))
