"""Sweep of the persistent encode -> Zinc COEFF pipeline (ZINC_TUNE_OVERLAP = 3)
against the PDL-chained serial path, from real slots on one GPU (C3 by default).
CUDA events, 3 warm-ups, median of 5.  Development tool, not the bench."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402
from sweep_zinc import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--variants", default="0,1,2")
    ap.add_argument("--enc", default="16,24,32,48,64,96")
    ap.add_argument("--ring", default="256")
    ap.add_argument("--mpc", default="2")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    B = args.batch or cfg.batch
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    _, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
    slots = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
    ct = ctx.empty_ct(B)
    by = B * (2 * cfg.L * cfg.n * 8 + slots[0].numel() * 8)
    peak = 6549.1

    def rep(name, ms, **kw):
        gbs = by / (ms / 1e3) / 1e9
        print(json.dumps({"case": name, "ms": ms, "ct_per_s": B / (ms / 1e3), "frac": gbs / peak, **kw}), flush=True)

    run = lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, slots, 1, 0, out=ct)  # noqa: E731
    rep("serial_pdl", timeit(run))
    ref = ct.clone()
    Z.tune(Z.TUNE_OVERLAP, 3)
    for v in [int(x) for x in args.variants.split(",")]:
        Z.tune(Z.TUNE_PIPE_VARIANT, v)
        for r in [int(x) for x in args.ring.split(",")]:
            Z.tune(Z.TUNE_ENCODE_CHUNK_BYTES, r * cfg.n * 8)
            for mpc in [int(x) for x in args.mpc.split(",")]:
                Z.tune(Z.TUNE_COEFF_MSGS_PER_CTA, mpc)
                for e in [int(x) for x in args.enc.split(",")]:
                    Z.tune(Z.TUNE_PIPE_ENC_CTAS, e)
                    ms = timeit(run)
                    ok = bool(torch.equal(ct, ref))
                    rep("pipe", ms, variant=v, ring=r, mpc=mpc, enc=e, equal=ok)
    Z.tune(Z.TUNE_OVERLAP, 0)
    Z.tune(Z.TUNE_COEFF_MSGS_PER_CTA, 2)
    Z.tune(Z.TUNE_ENCODE_CHUNK_BYTES, 32 << 20)


if __name__ == "__main__":
    main()
