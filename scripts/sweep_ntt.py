"""Throughput of the NTT-bound paths (Zinc NTT form, vanilla both forms, the
standalone forward/inverse NTT) from int64 plaintexts on one GPU, in
butterflies/s and as a fraction of the measured integer peak (K11).
CUDA events, 2 warm-ups, median of 5.  Development tool, not the bench."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, int_plaintexts  # noqa: E402


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


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    cfg = CONFIGS[name]
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.NTT)
    m = torch.from_numpy(int_plaintexts(cfg.log_n, 64, seed=1, bound_bits=44)).cuda().repeat(B // 64, 1)
    ct = ctx.empty_ct(B)
    sink = torch.zeros(2, dtype=torch.uint64, device="cuda")
    Z.zinc_int_peak(ctx, 148 * 8, 200, sink)
    ms = timeit(lambda: Z.zinc_int_peak(ctx, 148 * 8, 4000, sink), 3, 1)
    peak = 148 * 8 * 256 * 8 * 4000 / (ms / 1e3)
    half = cfg.n // 2 * cfg.log_n
    res = {"config": name, "batch": B, "int_peak_Gbfly": peak / 1e9}
    cases = [
        ("zinc_ntt", 2, lambda: Z.zinc_encrypt_batch(ctx, cache, Z.NTT, m, 1, 0, out=ct)),
        ("vanilla_ntt", 3, lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, m, 1, 0, out=ct)),
        ("vanilla_coeff", 3, lambda: Z.ckks_encrypt_batch(ctx, pk, Z.COEFF, m, 1, 0, out=ct)),
        ("ntt_fwd", 2, lambda: Z.zinc_ntt_forward(ctx, ct.view(-1, ctx.L, ctx.n))),
        ("ntt_inv", 2, lambda: Z.zinc_ntt_inverse(ctx, ct.view(-1, ctx.L, ctx.n))),
    ]
    for cname, transforms, fn in cases:
        t = timeit(fn)
        bf = transforms * cfg.L * half * B
        res[cname] = {"ms": t, "ct_per_s": B / (t / 1e3), "Gbfly": bf / (t / 1e3) / 1e9,
                      "frac_k11": bf / (t / 1e3) / peak}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
