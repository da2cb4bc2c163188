"""Small end-to-end run of every kernel for compute-sanitizer (one tool per
gpurun call): C1 (N=2^12) and a 2-message N=2^15 batch (the cluster-split
kernels), CKKS / BFV / BGV, both forms, encode / decrypt / decode, Eq. 2 kernels,
the PDL-chained encode -> path chunk pipelines.  Exits non-zero on any library error."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, int_plaintexts, slots_batch  # noqa: E402


def run(cfg, B, scheme=0, t=0):
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale, scheme=scheme, t=t)
    sk, _, pk = Z.zinc_keygen(ctx, 1)
    if scheme == 0:
        z = slots_batch(cfg, 0, B)
        if cfg.complex_slots:
            z = np.stack([z.real, z.imag], axis=-1)
        pt = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    else:
        pt = torch.from_numpy(int_plaintexts(cfg.log_n, B, 3) % t).cuda()
    for form in (Z.COEFF, Z.NTT):
        cache = Z.zinc_precompute_cache(ctx, pk, 2, form)
        for ct in (Z.zinc_encrypt_batch(ctx, cache, form, pt, 3, 0), Z.ckks_encrypt_batch(ctx, pk, form, pt, 3, 0)):
            coeff, st, _ = Z.ckks_decrypt_batch(ctx, sk, form, ct)
            assert int(st.sum()) == 0
            Z.zinc_ct_sum_batch(ctx, Z.zinc_ct_add_batch(ctx, ct, ct))
    if scheme == 0:
        for pdl in (0, 1):  # multi-chunk chains (double-buffered scratch), with and without PDL
            Z.tune(Z.TUNE_PDL, pdl)
            Z.tune(Z.TUNE_ENCODE_CHUNK_BYTES, 1 << 16)
            Z.tune(Z.TUNE_NTT_CHUNK_MSGS, 1)
            Z.zinc_encrypt_batch(ctx, Z.zinc_precompute_cache(ctx, pk, 2, Z.COEFF), Z.COEFF, pt, 3, 0)
            Z.ckks_encrypt_batch(ctx, pk, Z.NTT, pt, 3, 0)
        Z.tune(Z.TUNE_PDL, 1)
        Z.tune(Z.TUNE_ENCODE_CHUNK_BYTES, 32 << 20)
        Z.tune(Z.TUNE_NTT_CHUNK_MSGS, 0)
    torch.cuda.synchronize()
    ctx.close()


run(CONFIGS["C1"], 5)
run(CONFIGS["C1"], 3, scheme=1, t=65537)
run(CONFIGS["C1"], 3, scheme=2, t=65537)
run(CONFIGS["C4"], 2)
print("sanitize_small ok")
