"""Throughput of the transform-bound paths (Zinc NTT form, vanilla both forms,
decrypt, the standalone forward/inverse NTT) from int64 plaintexts on one GPU, in
butterflies/s and as a fraction of the measured integer peak (K11) of the
butterflies each path runs.  CUDA events, 2 warm-ups, median of 5.
Usage: python scripts/sweep_ntt.py [config] [batch] [case,...]   (development tool)"""
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


def k11(ctx, variant, sink):
    Z.zinc_int_peak(ctx, 148 * 8, 200, sink, variant=variant)
    ms = timeit(lambda: Z.zinc_int_peak(ctx, 148 * 8, 4000, sink, variant=variant), 3, 1)
    return 148 * 8 * 256 * 8 * 4000 / (ms / 1e3)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    only = set(sys.argv[3].split(",")) if len(sys.argv) > 3 else None
    cfg = CONFIGS[name]
    split = os.environ.get("ZINC_SPLIT")
    if split is not None:
        Z.tune(Z.TUNE_SPLIT, int(split))
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.NTT)
    m = torch.from_numpy(int_plaintexts(cfg.log_n, 64, seed=1, bound_bits=44)).cuda().repeat(B // 64, 1)
    ct = ctx.empty_ct(B)
    sink = torch.zeros(2, dtype=torch.uint64, device="cuda")
    nr_ok = max(ctx.q) < (1 << 58)
    peaks = {v: k11(ctx, v, sink) for v in (0, 1, 2, 3) if v != 1 or nr_ok}
    fwd = peaks[1] if nr_ok else peaks[2]      # the CKKS forward butterfly at this modulus
    half = cfg.n // 2 * cfg.log_n
    res = {"config": name, "batch": B, "split": split, "k11_Gbfly": {k: v / 1e9 for k, v in peaks.items()}}

    def mix(n_fwd, n_inv, fwd_peak):
        return (n_fwd + n_inv) / (n_fwd / fwd_peak + n_inv / peaks[3])

    ctc = ctx.empty_ct(B)
    Z.ckks_encrypt_batch(ctx, pk, Z.COEFF, m, 1, 0, out=ctc)
    cases = [
        ("zinc_ntt", 2, mix(2, 0, fwd), lambda: Z.zinc_encrypt_batch(ctx, cache, Z.NTT, m, 1, 0, out=ct)),
        ("vanilla_ntt", 3, mix(3, 0, fwd), lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, m, 1, 0, out=ct)),
        ("vanilla_coeff", 3, mix(1, 2, fwd), lambda: Z.ckks_encrypt_batch(ctx, pk, Z.COEFF, m, 1, 0, out=ct)),
        ("decrypt_coeff", 2, mix(1, 1, peaks[2]), lambda: Z.ckks_decrypt_batch(ctx, sk, Z.COEFF, ctc, slots=False)),
        ("ntt_fwd", 2, peaks[2], lambda: Z.zinc_ntt_forward(ctx, ct.view(-1, ctx.L, ctx.n))),
        ("ntt_inv", 2, peaks[3], lambda: Z.zinc_ntt_inverse(ctx, ct.view(-1, ctx.L, ctx.n))),
    ]
    for cname, transforms, peak, fn in cases:
        if only and cname not in only:
            continue
        t = timeit(fn)
        bf = transforms * cfg.L * half * B
        res[cname] = {"ms": t, "ct_per_s": B / (t / 1e3), "Gbfly": bf / (t / 1e3) / 1e9,
                      "peak_Gbfly": peak / 1e9, "frac": bf / (t / 1e3) / peak}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
