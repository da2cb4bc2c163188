"""Pins for the oracle's BFV / BGV variants (section 4.2).

Independent arithmetic: Delta = floor(Q/t) and the decryptions use Python big
integers (CRT written out here, not the oracle's); the zero-randomness hook is
checked against Delta * m computed in Python; correctness is the end-to-end
identity Dec(Enc(m)) = m of both schemes (Theorem 1's argument),
and the Zinc forms against vanilla with summed (t-scaled for BGV) errors.
"""
import numpy as np
import pytest

from workloads import CONFIGS

T_VALUES = [2, 17, 65537, (1 << 31) - 1]


def big_q(P):
    Q = 1
    for v in P.q:
        Q *= int(v)
    return Q


def py_crt_centered(P, xl):
    q = [int(v) for v in P.q]
    Q = big_q(P)
    out = []
    for j in range(P.n):
        x = 0
        for i, qi in enumerate(q):
            Mi = Q // qi
            x += int(xl[i][j]) * Mi * pow(Mi, -1, qi)
        x %= Q
        out.append(x - Q if x > Q // 2 else x)
    return out, Q


@pytest.fixture(scope="module")
def P(orc):
    c = CONFIGS["C1"]
    return orc.Params.make(c.log_n, c.bits, c.log_scale)


@pytest.mark.parametrize("t", T_VALUES)
def test_bfv_delta_residues_match_big_integers(orc, P, t):
    Q = big_q(P)
    assert orc.bfv_delta_mod(P, t) == [(Q // t) % int(q) for q in P.q]


@pytest.mark.parametrize("t", [17, 65537])
def test_bfv_zero_randomness_hook_is_delta_m(orc, P, t):
    """u = e1 = e2 = 0: c1 = Delta.m (COEFF form), c2 = 0 (SPEC.md:187 example, scaled up)."""
    rng = np.random.default_rng(1)
    m = rng.integers(-3 * t, 3 * t, P.n)           # any representative: the plaintext is m mod t
    _, _, pk = orc.keygen(P, 5)
    pt = orc.plaintext_residues(P, orc.BFV, t, m)
    zero = np.zeros(P.n, dtype=np.int64)
    ct = orc.encrypt_general_explicit(P, pk, pt, zero, zero, zero, 1, orc.COEFF)
    Q = big_q(P)
    want = np.array([[((Q // t) * (int(v) % t)) % int(q) for v in m] for q in P.q], dtype=np.uint64)
    assert np.array_equal(ct[0], want) and not ct[1].any()


@pytest.mark.parametrize("scheme", ["BFV", "BGV"])
@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("t", [17, 65537])
def test_decrypt_encrypt_identity_vanilla_and_zinc(orc, P, scheme, form, t):
    s = getattr(orc, scheme)
    sk, sk_ntt, pk = orc.keygen_scheme(P, 11, s, t)
    cache = orc.precompute_cache_scheme(P, s, t, pk, 12, form)
    rng = np.random.default_rng([t, form])
    for msg in range(3):
        m = rng.integers(0, t, P.n)
        for ct in (orc.encrypt_scheme(P, s, t, pk, m, 13, msg, form),
                   orc.zinc_encrypt_scheme(P, s, t, cache, form, m, 13, msg)):
            assert np.array_equal(orc.decrypt_scheme(P, s, t, sk_ntt, ct, form), m)


def test_decrypt_scheme_crt_matches_independent_crt(orc, P):
    t = 65537
    sk, sk_ntt, pk = orc.keygen_scheme(P, 3, orc.BFV, t)
    m = np.random.default_rng(2).integers(0, t, P.n)
    ct = orc.encrypt_scheme(P, orc.BFV, t, pk, m, 4, 0, orc.COEFF)
    _, _, xl = orc.decrypt(P, sk_ntt, ct, orc.COEFF, want_limbs=True)
    xs, Q = py_crt_centered(P, xl)
    # BFV residual: x - Delta m is the noise, far below Delta / 2
    D = Q // t
    def centred(v):
        v %= Q
        return v - Q if v > Q // 2 else v
    noise = max(abs(centred(x - D * int(v))) for x, v in zip(xs, m))
    assert noise < D // 1000


def test_bgv_key_error_is_t_scaled(orc, P):
    """Reading A17: [pk1 + pk2.sk]_Q = t.e (every coefficient a multiple of t, |e| <= 21)."""
    t = 65537
    sk, sk_ntt, pk = orc.keygen_scheme(P, 9, orc.BGV, t)
    # pk1 + pk2.sk in NTT form, back to coefficients, limb by limb
    x = np.zeros((P.L, P.n), dtype=np.uint64)
    for i, q in enumerate(P.q):
        q = int(q)
        x[i] = [(int(a) + int(b) * int(s)) % q for a, b, s in zip(pk[0][i], pk[1][i], sk_ntt[i])]
    orc_x = x.copy()
    from oracle import lib, _p, _u64p
    lib().orc_intt_limbs(_p(orc_x, _u64p), P.log_n, P.L, _p(P.q, _u64p), _p(P.psi, _u64p))
    xs, _ = py_crt_centered(P, orc_x)
    assert all(v % t == 0 and abs(v // t) <= 21 for v in xs)


@pytest.mark.parametrize("form", [0, 1])
def test_bgv_zinc_equals_vanilla_with_summed_scaled_errors(orc, P, form):
    """Zinc_BGV(m) = Vanilla_BGV(m; u*, e1* + e1', e2* + e2'): the cache's errors and the
    injected ones add before the t-scaling ("add t.e1' and t.e2'")."""
    t = 65537
    _, _, pk = orc.keygen_scheme(P, 21, orc.BGV, t)
    n = P.n
    u = orc.sample_ternary(22, orc.CACHE_MSG, orc.TAG_ENC_U, n)
    e1 = orc.sample_cbd(22, orc.CACHE_MSG, orc.TAG_ENC_E1, n)
    e2 = orc.sample_cbd(22, orc.CACHE_MSG, orc.TAG_ENC_E2, n)
    e1p = orc.sample_cbd(23, 5, orc.TAG_ZINC_E1, n)
    e2p = orc.sample_cbd(23, 5, orc.TAG_ZINC_E2, n)
    m = np.random.default_rng(3).integers(0, t, n)
    cache = orc.precompute_cache_scheme(P, orc.BGV, t, pk, 22, form)
    got = orc.zinc_encrypt_scheme(P, orc.BGV, t, cache, form, m, 23, 5)
    pt = orc.plaintext_residues(P, orc.BGV, t, m)
    want = orc.encrypt_general_explicit(P, pk, pt, u, e1 + e1p, e2 + e2p, t, form)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("scheme", ["BFV", "BGV"])
def test_additive_homomorphism_mod_t(orc, P, scheme):
    """Eq. 2: Dec(ct_a + ct_b) = m_a + m_b mod t."""
    t = 65537
    s = getattr(orc, scheme)
    sk, sk_ntt, pk = orc.keygen_scheme(P, 31, s, t)
    rng = np.random.default_rng(4)
    ma, mb = rng.integers(0, t, P.n), rng.integers(0, t, P.n)
    a = orc.encrypt_scheme(P, s, t, pk, ma, 32, 0, orc.COEFF)
    b = orc.encrypt_scheme(P, s, t, pk, mb, 32, 1, orc.COEFF)
    q = P.q.astype(object)[None, :, None]
    c = ((a.astype(object) + b.astype(object)) % q).astype(np.uint64)
    assert np.array_equal(orc.decrypt_scheme(P, s, t, sk_ntt, c, orc.COEFF), (ma + mb) % t)


def test_ckks_scheme_path_equals_plain_ckks(orc, P):
    """scheme 0 through the general entry points reproduces the CKKS oracle bit for bit."""
    _, _, pk = orc.keygen(P, 41)
    m = np.random.default_rng(5).integers(-(1 << 40), 1 << 40, P.n)
    for form in (0, 1):
        assert np.array_equal(orc.encrypt_scheme(P, orc.CKKS, 0, pk, m, 42, 7, form),
                              orc.vanilla_encrypt(P, pk, m, 42, 7, form))
        cache = orc.precompute_cache(P, pk, 43, form)
        assert np.array_equal(orc.precompute_cache_scheme(P, orc.CKKS, 0, pk, 43, form), cache)
        assert np.array_equal(orc.zinc_encrypt_scheme(P, orc.CKKS, 0, cache, form, m, 44, 8),
                              orc.zinc_encrypt(P, cache, form, m, 44, 8))
