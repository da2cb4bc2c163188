"""C2 Zinc COEFF from slots (4096 messages) step time + encode time, median of 5; plaintexts
compared with a reference file when given (development tool, A/B via ZINC_LIB_PATH)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402


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


cfg = CONFIGS["C2"]
B = 4096
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
_, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
zd = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
ct = ctx.empty_ct(B)
m = Z.ckks_encode_batch(ctx, zd)
ms = timeit(lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, 3, 0, out=ct))
enc = timeit(lambda: Z.ckks_encode_batch(ctx, zd, out=m))
byt = B * (2 * cfg.L * cfg.n * 8 + cfg.n * 8)
ref = sys.argv[1] if len(sys.argv) > 1 else None
same = None
if ref:
    if os.path.exists(ref):
        same = bool(torch.equal(torch.load(ref).cuda(), m))
    else:
        torch.save(m.cpu(), ref)
print(json.dumps({"lib": os.environ.get("ZINC_LIB_PATH", "default"), "ms": round(ms, 4),
                  "hbm_frac": round(byt / (ms * 1e-3) / 1e9 / 6547.2, 4), "encode_ms": round(enc, 4), "m_equal": same}))
