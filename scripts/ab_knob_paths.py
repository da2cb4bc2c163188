"""A/B of one tuning knob on the slots -> transform paths (Zinc NTT form, vanilla NTT form):
python scripts/ab_knob_paths.py KNOB V0 V1 [config] [batch].  Alternates the two values 3 times,
median of 3 each, and checks the ciphertexts are identical.  Development tool."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402


def timeit(fn, reps=3, warm=1):
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


knob, v0, v1 = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = CONFIGS[sys.argv[4] if len(sys.argv) > 4 else "C3"]
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
_, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.NTT)
B = int(sys.argv[5]) if len(sys.argv) > 5 else cfg.batch
z = slots_batch(cfg, 0, B)
if cfg.complex_slots:
    z = np.stack([z.real, z.imag], axis=-1)
slots = torch.from_numpy(np.ascontiguousarray(z)).cuda()
ct = ctx.empty_ct(B)
out = {"knob": knob, "config": cfg.name, "batch": B}
for name, fn in (("zinc_ntt", lambda: Z.zinc_encrypt_batch(ctx, cache, Z.NTT, slots, 1, 0, out=ct)),
                 ("vanilla_ntt", lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, slots, 1, 0, out=ct))):
    res = {v0: [], v1: []}
    outs = {}
    for _ in range(3):
        for v in (v0, v1):
            Z.tune(knob, v)
            res[v].append(timeit(fn))
            if v not in outs:
                outs[v] = ct.clone()
    out[name] = {str(v0): float(np.median(res[v0])), str(v1): float(np.median(res[v1])),
                 "ct_per_s": {str(v): B / float(np.median(res[v])) * 1e3 for v in (v0, v1)},
                 "equal": bool(torch.equal(outs[v0], outs[v1]))}
    del outs
print(json.dumps(out))
