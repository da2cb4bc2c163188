"""Edge cases of the launch geometry through the C ABI: single / tiny / ragged batches on every
path, message indices at the top of the 64-bit range, and the largest BASELINE batch (C5's
65536 messages, 128 GiB of ciphertexts) with sampled messages checked against the oracle."""
import numpy as np
import pytest
import torch

from workloads import CONFIGS, int_plaintexts

pytestmark = pytest.mark.gpu
NTT, COEFF = 0, 1


@pytest.fixture(scope="module")
def Z():
    import paper_2408_07304_b200 as Z
    return Z


@pytest.fixture(scope="module")
def c3(Z, orc):
    cfg = CONFIGS["C3"]
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    P = orc.Params.make(cfg.log_n, cfg.bits, cfg.log_scale)
    sk, _, pk = Z.zinc_keygen(ctx, 5)
    _, _, o_pk = orc.keygen(P, 5)
    caches = {f: Z.zinc_precompute_cache(ctx, pk, 6, f) for f in (NTT, COEFF)}
    o_caches = {f: orc.precompute_cache(P, o_pk, 6, f) for f in (NTT, COEFF)}
    return ctx, P, pk, o_pk, caches, o_caches


@pytest.mark.parametrize("B", [1, 2, 3, 5])
@pytest.mark.parametrize("path", ["zinc", "vanilla"])
@pytest.mark.parametrize("form", [NTT, COEFF])
def test_tiny_batches_every_path(Z, orc, c3, B, path, form):
    ctx, P, pk, o_pk, caches, o_caches = c3
    m = int_plaintexts(P.log_n, B, seed=B, bound_bits=44)
    base = (1 << 64) - 1 - 8  # message indices up to 2^64 - 2: the counter's top words all set
    md = torch.from_numpy(m).cuda()
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(ctx, caches[form], form, md, 9, base)
    else:
        ct = Z.ckks_encrypt_batch(ctx, pk, form, md, 9, base)
    got = ct.cpu().numpy()
    b = B - 1
    want = (orc.zinc_encrypt(P, o_caches[form], form, m[b], 9, base + b) if path == "zinc"
            else orc.vanilla_encrypt(P, o_pk, m[b], 9, base + b, form))
    assert np.array_equal(got[b], want)


def test_largest_baseline_batch_c5_65536(Z, orc):
    """C5's largest batch in one call: 65536 messages -> 128 GiB of ciphertexts on one GPU."""
    cfg = CONFIGS["C5"]
    B = 65536
    torch.cuda.empty_cache()
    need = B * (2 * cfg.L * cfg.n * 8 + cfg.n * 8)
    if torch.cuda.mem_get_info()[0] < need * 1.05:
        pytest.skip("not enough free device memory for the 65536-message batch")
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
    P = orc.Params.make(cfg.log_n, cfg.bits, cfg.log_scale)
    sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, COEFF)
    gen = torch.Generator(device="cuda").manual_seed(11)
    m = torch.randint(-(1 << 44), 1 << 44, (B, cfg.n), dtype=torch.int64, device="cuda", generator=gen)
    ct = Z.zinc_encrypt_batch(ctx, cache, COEFF, m, cfg.enc_seed, 0)
    torch.cuda.synchronize()
    idx = [0, 1, 40000, B - 1]
    got = {b: ct[b].cpu().numpy() for b in idx}
    mm = {b: m[b].cpu().numpy() for b in idx}
    del ct, m
    torch.cuda.empty_cache()
    _, _, o_pk = orc.keygen(P, cfg.key_seed)
    o_cache = orc.precompute_cache(P, o_pk, cfg.cache_seed, COEFF)
    for b in idx:
        assert np.array_equal(got[b], orc.zinc_encrypt(P, o_cache, COEFF, mm[b], cfg.enc_seed, b)), b
