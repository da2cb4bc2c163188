"""Per-kernel breakdown of one full-batch call from slots (device time with CUDA events around
the call; the library's traced per-kernel sums) and the step-level HBM fraction of Zinc COEFF
form.  python scripts/breakdown.py [config,...] [path,...]   (development tool)"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6549.1
res = {}
for kv in os.environ.get("ZINC_KNOBS", "").split(","):
    if kv:
        k, v = kv.split("=")
        Z.tune(int(k), int(v))
for name in (sys.argv[1] if len(sys.argv) > 1 else "C2,C3,C4").split(","):
    cfg = CONFIGS[name]
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
    B = cfg.batch
    z = slots_batch(cfg, 0, B)
    if cfg.complex_slots:
        z = np.stack([z.real, z.imag], axis=-1)
    zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    ct = ctx.empty_ct(B)
    fn = lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, 1, 0, out=ct)
    for _ in range(3):
        fn()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    Z.profile_enable(True)
    fn()
    torch.cuda.synchronize()
    prof = {k: {"ms": round(v[0], 4), "launches": v[1]} for k, v in Z.profile_read().items()}
    Z.profile_enable(False)
    ms = statistics.median(ts)
    per_ct = 2 * cfg.L * cfg.n * 8 + (cfg.n * 8 if cfg.complex_slots else cfg.n // 2 * 8)
    res[name] = {"batch": B, "ms": ms, "ct_per_s": B / ms * 1e3, "hbm_frac_step": B * per_ct / (ms / 1e3) / 1e9 / peak,
                 "kernels": prof}
    del ct, zd
    ctx.close()
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
