"""Pins for the oracle's scheme layer: keygen (Eq. 7), vanilla (Eq. 8, reading A1),
cache, Zinc (Algorithm 1, Eq. 4 + Eq. 9), decryption (Eq. 10) and
Theorem 1's residual, Eq. 2 homomorphism, and the transform accounting of
PAPER.md:308-317.

Independent arithmetic: products of a ternary polynomial with a residue vector
are computed by signed negacyclic shifts in numpy (no NTT); products of small
integer polynomials by numpy.convolve, folded negacyclically.
"""
import numpy as np
import pytest

from workloads import CONFIGS

C1 = CONFIGS["C1"]


def negacyclic_int(a, b):
    """Exact product of two small integer polynomials in Z[X]/(X^N+1)."""
    n = len(a)
    full = np.convolve(np.asarray(a, dtype=np.int64), np.asarray(b, dtype=np.int64))
    out = full[:n].copy()
    out[: n - 1] -= full[n:]
    return out


def ternary_times_residues(t, a, q):
    """(t * a) mod q with t ternary (int) and a canonical residues < q < 2^62,
    by sum of +-X^i a over the support of t (negacyclic shifts)."""
    n = len(a)
    a = np.asarray(a, dtype=np.uint64)
    acc = np.zeros(n, dtype=np.uint64)
    q = np.uint64(q)
    for i in np.nonzero(t)[0]:
        # X^i a: coefficients shift up by i, the wrapped ones change sign
        sh = np.empty(n, dtype=np.uint64)
        sh[i:] = a[: n - i]
        wrapped = a[n - i:]
        sh[:i] = np.where(wrapped == 0, 0, q - wrapped)
        if t[i] < 0:
            sh = np.where(sh == 0, 0, q - sh)
        acc = (acc + sh) % q
    return acc


def residues(v, q):
    return (np.asarray(v, dtype=object) % int(q)).astype(np.uint64)


@pytest.fixture(scope="module")
def small(orc):
    """N = 256, three limbs (limb 0 largest), Delta = 2^25."""
    P = orc.Params.make(8, [45, 36, 36], 25)
    sk, sk_ntt, pk = orc.keygen(P, 77)
    return P, sk, sk_ntt, pk


@pytest.fixture(scope="module")
def c1(orc):
    P = orc.Params.make(C1.log_n, C1.bits, C1.log_scale)
    sk, sk_ntt, pk = orc.keygen(P, C1.key_seed)
    return P, sk, sk_ntt, pk


def test_keygen_eq7(orc, small):
    """[pk1 + pk2 . sk]_q = e exactly (Eq. 7), so its infinity norm is <= 21."""
    P, sk, sk_ntt, pk = small
    assert set(np.unique(sk).tolist()) <= {-1, 0, 1}
    e = orc.sample_cbd(77, 0, orc.TAG_PK_E, P.n)
    pk_c = orc.intt_limbs(P, pk[0])
    pk2_c = orc.intt_limbs(P, pk[1])
    for i, qi in enumerate(map(int, P.q)):
        lhs = (pk_c[i] + ternary_times_residues(sk, pk2_c[i], qi)) % np.uint64(qi)
        assert np.array_equal(lhs, residues(e, qi))
        # pk2 = a is the uniform draw of limb i (C-5)
        assert np.array_equal(pk2_c[i], orc.sample_uniform(77, 0, orc.TAG_PK_A, i, qi, P.n))
        assert np.array_equal(sk_ntt[i], orc.ntt(residues(sk, qi), P.log_n, qi, int(P.psi[i])))


@pytest.mark.parametrize("form", [0, 1])
def test_vanilla_zero_randomness(orc, small, form):
    """u = e1 = e2 = 0 gives ct = (m, 0)."""
    P, sk, sk_ntt, pk = small
    m = np.random.default_rng(1).integers(-2**40, 2**40, P.n)
    z = np.zeros(P.n, dtype=np.int64)
    ct = orc.vanilla_encrypt_explicit(P, pk, m, z, z, z, form)
    for i, qi in enumerate(map(int, P.q)):
        mi = residues(m, qi)
        assert np.array_equal(ct[0, i], mi if form == 1 else orc.ntt(mi, P.log_n, qi, int(P.psi[i])))
        assert (ct[1, i] == 0).all()


@pytest.mark.parametrize("form", [0, 1])
def test_vanilla_theorem1_residual(orc, small, form):
    """Dec(Enc(m)) - m = e.u + e1 + e2.sk exactly (Theorem 1 algebra, PAPER.md:242-248,
    with e1' = e2' = 0), on every limb; CRT status 0."""
    P, sk, sk_ntt, pk = small
    seed, msg = 4242, 17
    m = np.random.default_rng(2).integers(-2**30, 2**30, P.n)
    ct = orc.vanilla_encrypt(P, pk, m, seed, msg, form)
    x, st, xl = orc.decrypt(P, sk_ntt, ct, form, want_limbs=True)
    e = orc.sample_cbd(77, 0, orc.TAG_PK_E, P.n)
    u = orc.sample_ternary(seed, msg, orc.TAG_ENC_U, P.n)
    e1 = orc.sample_cbd(seed, msg, orc.TAG_ENC_E1, P.n)
    e2 = orc.sample_cbd(seed, msg, orc.TAG_ENC_E2, P.n)
    v = negacyclic_int(e, u) + e1 + negacyclic_int(e2, sk)
    assert st == 0
    assert np.array_equal(x - m, v)
    for i, qi in enumerate(map(int, P.q)):
        assert np.array_equal(xl[i], residues(m + v, qi))
    # worst-case bound 21 (2N + 1) (SPEC.md:222 restated for CBD)
    assert np.abs(v).max() <= 21 * (2 * P.n + 1)


@pytest.mark.parametrize("form", [0, 1])
def test_zinc_equals_vanilla_with_summed_errors(orc, small, form):
    """Zinc(m) is bit-identical to vanilla(m; u*, e1* + e1', e2* + e2')."""
    P, sk, sk_ntt, pk = small
    cseed, seed, msg = 999, 31337, 5
    cache = orc.precompute_cache(P, pk, cseed, form)
    m = np.random.default_rng(3).integers(-2**35, 2**35, P.n)
    ct = orc.zinc_encrypt(P, cache, form, m, seed, msg)
    us = orc.sample_ternary(cseed, orc.CACHE_MSG, orc.TAG_ENC_U, P.n)
    e1s = orc.sample_cbd(cseed, orc.CACHE_MSG, orc.TAG_ENC_E1, P.n)
    e2s = orc.sample_cbd(cseed, orc.CACHE_MSG, orc.TAG_ENC_E2, P.n)
    e1p = orc.sample_cbd(seed, msg, orc.TAG_ZINC_E1, P.n)
    e2p = orc.sample_cbd(seed, msg, orc.TAG_ZINC_E2, P.n)
    ref = orc.vanilla_encrypt_explicit(P, pk, m, us, e1s + e1p, e2s + e2p, form)
    assert np.array_equal(ct, ref)
    # the cache is Enc(0) with the cache stream (C-8)
    z = np.zeros(P.n, dtype=np.int64)
    assert np.array_equal(cache, orc.vanilla_encrypt_explicit(P, pk, z, us, e1s, e2s, form))
    assert np.array_equal(ct, orc.zinc_encrypt_explicit(P, cache, form, m, e1p, e2p))


def test_zinc_coeff_difference_is_the_injected_error(orc, small):
    """COEFF form: ct - cache - (m, 0) = (e1', e2') exactly (Eq. 4 + Eq. 9)."""
    P, sk, sk_ntt, pk = small
    cache = orc.precompute_cache(P, pk, 1, 1)
    m = np.random.default_rng(4).integers(-2**35, 2**35, P.n)
    ct = orc.zinc_encrypt(P, cache, 1, m, 2, 3)
    e1p = orc.sample_cbd(2, 3, orc.TAG_ZINC_E1, P.n)
    e2p = orc.sample_cbd(2, 3, orc.TAG_ZINC_E2, P.n)
    for i, qi in enumerate(map(int, P.q)):
        d1 = (ct[0, i].astype(object) - cache[0, i].astype(object) - m) % qi
        d2 = (ct[1, i].astype(object) - cache[1, i].astype(object)) % qi
        assert np.array_equal(d1.astype(np.uint64), residues(e1p, qi))
        assert np.array_equal(d2.astype(np.uint64), residues(e2p, qi))


def test_forms_related_by_one_ntt(orc, small):
    """NTT(COEFF-form ct) == NTT-form ct for both paths."""
    P, sk, sk_ntt, pk = small
    m = np.random.default_rng(5).integers(-2**30, 2**30, P.n)
    for path in ("vanilla", "zinc"):
        if path == "vanilla":
            a = orc.vanilla_encrypt(P, pk, m, 7, 8, 1)
            b = orc.vanilla_encrypt(P, pk, m, 7, 8, 0)
        else:
            a = orc.zinc_encrypt(P, orc.precompute_cache(P, pk, 9, 1), 1, m, 7, 8)
            b = orc.zinc_encrypt(P, orc.precompute_cache(P, pk, 9, 0), 0, m, 7, 8)
        for c in range(2):
            assert np.array_equal(orc.ntt_limbs(P, a[c]), b[c])


def test_two_zinc_encryptions_differ_by_binomial84(orc, small):
    """SPEC.md:274, 436 adapted: two Zinc encryptions of one m differ by
    e' - e'' ~ Binomial(84, 1/2) - 42 per coefficient, |.| <= 42."""
    P, sk, sk_ntt, pk = small
    cache = orc.precompute_cache(P, pk, 1, 1)
    m = np.zeros(P.n, dtype=np.int64)
    diffs = []
    for msg in range(40):
        a = orc.zinc_encrypt(P, cache, 1, m, 11, 2 * msg)
        b = orc.zinc_encrypt(P, cache, 1, m, 11, 2 * msg + 1)
        assert not np.array_equal(a[0], b[0]) and not np.array_equal(a[1], b[1])
        q0 = int(P.q[0])
        d = (a[:, 0].astype(object) - b[:, 0].astype(object)) % q0
        d = np.where(d > q0 // 2, d - q0, d).astype(np.int64)
        diffs.append(d.ravel())
    d = np.concatenate(diffs)
    assert np.abs(d).max() <= 42
    assert abs(d.var() - 21.0) / 21.0 < 0.05
    assert abs(d.mean()) < 4 * np.sqrt(21.0 / len(d))


@pytest.mark.parametrize("form", [0, 1])
def test_theorem1_end_to_end_c1(orc, c1, form):
    """Theorem 1 + decode tolerance at C1 (Delta = 2^30 -> 1e-3, BASELINE.json)."""
    from workloads import message_slots
    P, sk, sk_ntt, pk = c1
    cache = orc.precompute_cache(P, pk, C1.cache_seed, form)
    for b in range(3):
        z = message_slots(C1, b)
        m = orc.encode(z, P.log_n, P.log_scale)
        for ct in (orc.zinc_encrypt(P, cache, form, m, C1.enc_seed, b),
                   orc.vanilla_encrypt(P, pk, m, C1.enc_seed, b, form)):
            x, st = orc.decrypt(P, sk_ntt, ct, form)
            assert st == 0
            assert np.max(np.abs(orc.decode(x, P.log_n, P.log_scale) - z)) < C1.tolerance()


def test_eq2_additive_homomorphism(orc, c1):
    """Eq. 2: Dec(Enc(a) + Enc(b)) ~ a + b within 2x tolerance."""
    from workloads import message_slots
    P, sk, sk_ntt, pk = c1
    cache = orc.precompute_cache(P, pk, C1.cache_seed, 1)
    za, zb = message_slots(C1, 10), message_slots(C1, 11)
    ca = orc.zinc_encrypt(P, cache, 1, orc.encode(za, P.log_n, P.log_scale), 5, 10)
    cb = orc.vanilla_encrypt(P, pk, orc.encode(zb, P.log_n, P.log_scale), 5, 11, 1)
    q = P.q.reshape(1, -1, 1)
    s = (ca + cb) % q   # residues < 2^36, no overflow
    x, st = orc.decrypt(P, sk_ntt, s, 1)
    assert st == 0
    assert np.max(np.abs(orc.decode(x, P.log_n, P.log_scale) - (za + zb))) < 2 * C1.tolerance()


def test_decrypt_wrong_key_fails_crt(orc, c1):
    P, sk, sk_ntt, pk = c1
    m = np.zeros(P.n, dtype=np.int64)
    ct = orc.vanilla_encrypt(P, pk, m, 1, 1, 1)
    other = orc.keygen(P, 12345)[1]
    x, st = orc.decrypt(P, other, ct, 1)
    assert st == 1


def test_noise_variance_closed_forms(orc, c1):
    """variance over coefficients, conditioned on the key:
    vanilla ~ (2/3)|e|^2 + 10.5 |s|^2 + 10.5, Zinc ~ (2/3)|e|^2 + 21 |s|^2 + 21,
    within 5 % averaged over 8 ciphertexts at N = 4096."""
    P, sk, sk_ntt, pk = c1
    e = orc.sample_cbd(C1.key_seed, 0, orc.TAG_PK_E, P.n)
    e2n, s2n = float((e.astype(np.float64) ** 2).sum()), float((sk.astype(np.float64) ** 2).sum())
    want_v = (2 / 3) * e2n + 10.5 * s2n + 10.5
    want_z = (2 / 3) * e2n + 21 * s2n + 21
    cache = orc.precompute_cache(P, pk, C1.cache_seed, 1)
    m = np.zeros(P.n, dtype=np.int64)
    var_v = np.mean([orc.decrypt(P, sk_ntt, orc.vanilla_encrypt(P, pk, m, 3, b, 1), 1)[0].astype(np.float64).var()
                     for b in range(8)])
    var_z = np.mean([orc.decrypt(P, sk_ntt, orc.zinc_encrypt(P, cache, 1, m, 3, b), 1)[0].astype(np.float64).var()
                     for b in range(8)])
    assert abs(var_v - want_v) / want_v < 0.05
    assert abs(var_z - want_z) / want_z < 0.05


def test_transform_accounting(orc, small):
    """vanilla = 3 transforms + 2 pointwise products per limb;
    Zinc COEFF = none; Zinc NTT = the errors' DFTs (+ the plaintext's own NTT)."""
    P, sk, sk_ntt, pk = small
    m = np.zeros(P.n, dtype=np.int64)
    for form in (0, 1):
        orc.counters_reset()
        orc.vanilla_encrypt(P, pk, m, 1, 1, form)
        assert orc.counters() == (3 * P.L, 2 * P.L * P.n)
    cache_c = orc.precompute_cache(P, pk, 1, 1)
    cache_n = orc.precompute_cache(P, pk, 1, 0)
    orc.counters_reset()
    orc.zinc_encrypt(P, cache_c, 1, m, 1, 1)
    assert orc.counters() == (0, 0)
    orc.counters_reset()
    orc.zinc_encrypt(P, cache_n, 0, m, 1, 1)
    assert orc.counters() == (3 * P.L, 0)


def test_ct_add_and_sum_match_big_integer_sums(orc, small):
    """orc_ct_add / orc_ct_sum against Python big-integer sums reduced mod q_i."""
    P = small[0]
    rng = np.random.default_rng(12)
    cts = np.stack([np.stack([np.stack([rng.integers(0, int(q), P.n, dtype=np.uint64) for q in P.q])
                              for _ in range(2)]) for _ in range(5)])
    q = np.array([int(v) for v in P.q], dtype=object)[None, None, :, None]
    add = (cts[:2].astype(object) + cts[2:4].astype(object)) % q
    assert np.array_equal(orc.ct_add(P, cts[:2], cts[2:4]), add.astype(np.uint64))
    tot = cts.astype(object).sum(axis=0) % q[0]
    assert np.array_equal(orc.ct_sum(P, cts), tot.astype(np.uint64))


def test_aggregation_decrypts_to_the_slot_sum(orc, c1):
    """Eq. 2 repeated: Dec(sum of k Zinc encryptions) = sum of the k plaintexts + noise."""
    P, sk, sk_ntt, pk = c1
    from workloads import slots_batch
    cache = orc.precompute_cache(P, pk, 3, orc.COEFF)
    z = slots_batch(C1, 0, 6)
    cts = np.stack([orc.zinc_encrypt(P, cache, orc.COEFF, orc.encode(z[k], P.log_n, P.log_scale), 4, k)
                    for k in range(6)])
    x, st = orc.decrypt(P, sk_ntt, orc.ct_sum(P, cts), orc.COEFF)
    assert st == 0
    err = np.max(np.abs(orc.decode(x, P.log_n, P.log_scale) - z.sum(axis=0)))
    assert err < 6 * C1.tolerance()
