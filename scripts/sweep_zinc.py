"""Launch-geometry sweep of the COEFF-form Zinc path on one GPU (C3 by default).

Times, with CUDA events on the launching stream (3 warm-ups, median of 5):
  encode alone, Zinc from int64 plaintexts (the kernel alone) and Zinc from
  slots (encode + kernel, overlapped or serial) for several tuning-knob values.
Prints one JSON line per measurement.  A development tool, not the bench."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402


def timeit(fn, reps=5, warm=3):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--mpc", default="1,2,4,8,16")
    ap.add_argument("--chunks-mb", default="16,32,48")
    ap.add_argument("--pads-kb", default="0,12")
    ap.add_argument("--pdl", default="1,0")
    ap.add_argument("--overlaps", default="0,1,2")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    B = args.batch or cfg.batch
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
    z = slots_batch(cfg, 0, B)
    slots = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    m = Z.ckks_encode_batch(ctx, slots)
    ct = ctx.empty_ct(B)
    ct_bytes = 2 * cfg.L * cfg.n * 8
    in_bytes = slots[0].numel() * 8
    peak = 6549.1

    def rep(name, ms, bytes_per_msg, **kw):
        gbs = B * bytes_per_msg / (ms / 1e3) / 1e9
        print(json.dumps({"case": name, "ms": ms, "ct_per_s": B / (ms / 1e3), "GBs": gbs, "frac": gbs / peak, **kw}),
              flush=True)

    rep("encode", timeit(lambda: Z.ckks_encode_batch(ctx, slots, out=m)), in_bytes + cfg.n * 8)
    for pdl in [int(x) for x in args.pdl.split(",")]:
      Z.tune(Z.TUNE_PDL, pdl)
      for pad in [int(x) for x in args.pads_kb.split(",")]:
          Z.tune(Z.TUNE_COEFF_SMEM_PAD, pad << 10)
          for mpc in [int(x) for x in args.mpc.split(",")]:
              Z.tune(Z.TUNE_COEFF_MSGS_PER_CTA, mpc)
              rep("zinc_i64", timeit(lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, m, 1, 0, out=ct)),
                  ct_bytes + cfg.n * 8, mpc=mpc, pad_kb=pad, pdl=pdl)
          for ov in [int(x) for x in args.overlaps.split(",")]:
              Z.tune(Z.TUNE_OVERLAP, ov)
              for mb in [int(x) for x in args.chunks_mb.split(",")]:
                  Z.tune(Z.TUNE_ENCODE_CHUNK_BYTES, mb << 20)
                  for mpc in [int(x) for x in args.mpc.split(",")]:
                      Z.tune(Z.TUNE_COEFF_MSGS_PER_CTA, mpc)
                      rep("zinc_slots", timeit(lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, slots, 1, 0, out=ct)),
                          ct_bytes + in_bytes, mpc=mpc, overlap=ov, chunk_mb=mb, pad_kb=pad, pdl=pdl)
    Z.tune(Z.TUNE_COEFF_SMEM_PAD, 0)
    # correctness spot check against the serial path
    Z.tune(Z.TUNE_OVERLAP, 0)
    ref = Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, slots[:600], 1, 0)
    Z.tune(Z.TUNE_OVERLAP, 1)
    Z.tune(Z.TUNE_ENCODE_CHUNK_BYTES, 16 << 20)
    got = Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, slots[:600], 1, 0)
    print(json.dumps({"case": "overlap_equals_serial", "ok": bool(torch.equal(ref, got))}), flush=True)


if __name__ == "__main__":
    main()
