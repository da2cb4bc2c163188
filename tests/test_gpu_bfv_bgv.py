"""GPU parity of the BFV (Eq. 12) and BGV (Eq. 13) variants (PAPER.md:319-343,
SURVEY.md 8(f) f2) against the oracle: keys, caches and ciphertexts bit-exact,
decryption = the plaintext mod t (and = the oracle's big-integer decryption)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

NTT, COEFF = 0, 1
CASES = [  # (name, log_n, bits, t)
    ("small", 12, [36, 36, 36], 65537),
    ("c3", 14, [54] * 8, 65537),
    ("c3_bigt", 14, [54] * 8, (1 << 31) - 1),
    ("c4", 15, [55] * 16, 786433),
]


@pytest.fixture(scope="module")
def Z():
    import paper_2408_07304_b200 as Z
    return Z


_cache = {}


def setup(Z, orc, case, scheme):
    key = (case, scheme)
    if key not in _cache:
        name, log_n, bits, t = [c for c in CASES if c[0] == case][0]
        ctx = Z.Context(log_n, bits, 0, scheme=scheme, t=t)
        P = orc.Params.make(log_n, bits, 20)
        sk, skc, pk = Z.zinc_keygen(ctx, 101)
        o = orc.keygen_scheme(P, 101, scheme, t)
        caches = {f: Z.zinc_precompute_cache(ctx, pk, 102, f) for f in (NTT, COEFF)}
        _cache[key] = (ctx, P, t, sk, pk, o, caches)
    return _cache[key]


@pytest.mark.parametrize("case", [c[0] for c in CASES])
@pytest.mark.parametrize("scheme", [1, 2])
def test_keys_and_caches_bit_exact(Z, orc, case, scheme):
    ctx, P, t, sk, pk, (o_sk, o_sk_ntt, o_pk), caches = setup(Z, orc, case, scheme)
    assert np.array_equal(sk.cpu().numpy(), o_sk_ntt)
    assert np.array_equal(pk.cpu().numpy(), o_pk)
    for f in (NTT, COEFF):
        want = orc.precompute_cache_scheme(P, scheme, t, o_pk, 102, f)
        assert np.array_equal(caches[f].cpu().numpy(), want), f


@pytest.mark.parametrize("case", ["small", "c3", "c3_bigt", "c4"])
@pytest.mark.parametrize("scheme", [1, 2])
@pytest.mark.parametrize("path", ["zinc", "vanilla"])
@pytest.mark.parametrize("form", [NTT, COEFF])
def test_encrypt_bit_exact_and_decrypt(Z, orc, case, scheme, path, form):
    ctx, P, t, sk, pk, (o_sk, o_sk_ntt, o_pk), caches = setup(Z, orc, case, scheme)
    B = 9
    rng = np.random.default_rng([scheme, form, len(path)])
    m = rng.integers(-2 * t, 2 * t, (B, P.n))          # any representative of m mod t
    m[0, :3] = [np.iinfo(np.int64).min, np.iinfo(np.int64).max, -1]
    md = torch.from_numpy(m).cuda()
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(ctx, caches[form], form, md, 7, 40)
        o_cache = orc.precompute_cache_scheme(P, scheme, t, o_pk, 102, form)
    else:
        ct = Z.ckks_encrypt_batch(ctx, pk, form, md, 7, 40)
    got = ct.cpu().numpy()
    for b in (0, 4, B - 1):
        if path == "zinc":
            want = orc.zinc_encrypt_scheme(P, scheme, t, o_cache, form, m[b], 7, 40 + b)
        else:
            want = orc.encrypt_scheme(P, scheme, t, o_pk, m[b], 7, 40 + b, form)
        assert np.array_equal(got[b], want), b
    coeff, status, slots = Z.ckks_decrypt_batch(ctx, sk, form, ct)
    assert slots is None and (status.cpu().numpy() == 0).all()
    dec = coeff.cpu().numpy()
    assert np.array_equal(dec, np.mod(m, t))
    if case == "small":
        assert np.array_equal(dec[4], orc.decrypt_scheme(P, scheme, t, o_sk_ntt, got[4], form))


def test_bfv_bgv_reject_slots_and_bad_moduli(Z, orc):
    ctx = setup(Z, orc, "small", 1)[0]
    z = torch.zeros((1, ctx.n // 2), dtype=torch.float64, device="cuda")
    with pytest.raises(Z.ZincError):
        Z.zinc_encrypt_batch(ctx, setup(Z, orc, "small", 1)[6][COEFF], COEFF, z, 1)
    for bad_t in (0, 1, 1 << 32):
        with pytest.raises(Z.ZincError):
            Z.Context(12, [36, 36, 36], 0, scheme=1, t=bad_t)


def test_bgv_homomorphic_sum_decrypts_mod_t(Z, orc):
    """Eq. 2 on the GPU ciphertexts: Dec(ct_a + ct_b) = m_a + m_b mod t (the sum itself
    formed here with torch integer ops; the decryption runs in the library)."""
    ctx, P, t, sk, pk, o, caches = setup(Z, orc, "c3", 2)
    rng = np.random.default_rng(8)
    ma, mb = rng.integers(0, t, (4, P.n)), rng.integers(0, t, (4, P.n))
    a = Z.zinc_encrypt_batch(ctx, caches[COEFF], COEFF, torch.from_numpy(ma).cuda(), 3, 0)
    b = Z.zinc_encrypt_batch(ctx, caches[COEFF], COEFF, torch.from_numpy(mb).cuda(), 3, 100)
    q = torch.tensor([int(v) for v in P.q], dtype=torch.float64)
    s = a.cpu().numpy().astype(object) + b.cpu().numpy().astype(object)
    s = (s % np.array([int(v) for v in P.q], dtype=object)[None, None, :, None]).astype(np.uint64)
    coeff, status, _ = Z.ckks_decrypt_batch(ctx, sk, COEFF, torch.from_numpy(s).cuda())
    assert (status.cpu().numpy() == 0).all()
    assert np.array_equal(coeff.cpu().numpy(), (ma + mb) % t)
