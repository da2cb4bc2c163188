"""Per-kernel device times (library tracing, CUDA events on the launch stream)
of one Zinc-from-slots call at several encode chunk sizes.  Development tool."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
B = cfg.batch
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
slots = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
ct = ctx.empty_ct(B)
m = Z.ckks_encode_batch(ctx, slots)
Z.tune(Z.TUNE_COEFF_MSGS_PER_CTA, 2)
for ov in (0, 1):
    Z.tune(Z.TUNE_OVERLAP, ov)
    for mb in (8, 32):
        Z.tune(Z.TUNE_ENCODE_CHUNK_BYTES, mb << 20)
        for _ in range(2):
            Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, slots, 1, 0, out=ct)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        Z.profile_enable(True)
        a.record()
        Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, slots, 1, 0, out=ct)
        b.record()
        torch.cuda.synchronize()
        prof = Z.profile_read()
        Z.profile_enable(False)
        print(json.dumps({"overlap": ov, "chunk_mb": mb, "total_ms": a.elapsed_time(b),
                          "kernels": {k: {"ms": v[0], "n": v[1], "us_per_launch": 1e3 * v[0] / v[1]}
                                      for k, v in prof.items()}}), flush=True)
# encode alone at several batch sizes (per-CTA latency vs throughput)
for nb in (64, 148, 256, 444, 1024, 4096):
    for _ in range(2):
        Z.ckks_encode_batch(ctx, slots[:nb], out=m[:nb])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        Z.ckks_encode_batch(ctx, slots[:nb], out=m[:nb])
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"encode_batch": nb, "us_per_call": 100 * a.elapsed_time(b)}), flush=True)
for nb in (64, 256, 1024):
    for _ in range(2):
        Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, m[:nb], 1, 0, out=ct[:nb])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, m[:nb], 1, 0, out=ct[:nb])
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"zinc_i64_batch": nb, "us_per_call": 100 * a.elapsed_time(b)}), flush=True)
