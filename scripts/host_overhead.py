"""Host-side cost of one API call (C5 batch 1): wall time from entering the Python call to its
return (the kernels are enqueued, not finished), split into the binding's marshalling and the
C call, with the GPU idle before each call.  python scripts/host_overhead.py  (development tool)"""
import ctypes
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

cfg = CONFIGS["C5"]
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
_, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
z = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, 1))).cuda()
ct = ctx.empty_ct(1)
L = Z.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = (ctx.handle, ctypes.c_void_p(cache.data_ptr()), Z.COEFF, 1, ctypes.c_void_p(z.data_ptr()), 1, 3, 0,
        ctypes.c_void_p(ct.data_ptr()), s)
res = {}
for name, fn in (("python_call", lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, z, 3, 0, out=ct)),
                 ("c_call", lambda: L.zinc_encrypt_batch(*args))):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        ts.append((t1 - t0) * 1e6)
    res[name] = {"median_us": round(statistics.median(ts), 2), "min_us": round(min(ts), 2)}
print(res)
