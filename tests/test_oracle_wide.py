"""Pins for the oracle's wide-plaintext path (the paper's own
parameters: N = 2^15, 15 x 55-bit primes + one 56-bit prime
(881-bit Q), Delta = 2^55).  At these scales |m_j| passes 2^63, so coefficients
are 128-bit integers and decryption needs a CRT beyond limb 0.

Independent arithmetic: closed forms in Python integers; the two-limb CRT is
checked against the full big-integer CRT; encryption against Enc(0) + m."""
import numpy as np
import pytest

PAPER_BITS = [56] + [55] * 15


@pytest.fixture(scope="module")
def P(orc):
    return orc.Params.make(15, PAPER_BITS, 55)


def test_paper_modulus_is_881_bits(orc, P):
    Q = 1
    for q in P.q:
        Q *= int(q)
    assert Q.bit_length() == 881 and int(P.q[0]) == max(int(q) for q in P.q)


@pytest.mark.parametrize("c", [300.25, -(2.0 ** 31) + 0.5, 123456789.0])
def test_wide_encode_constant_slots_closed_form(orc, c):
    """All slots = c  =>  m = round(Delta c) X^0 exactly, beyond 2^63 (C-6 closed form)."""
    log_n, ls = 15, 55
    z = np.full(1 << (log_n - 1), c)
    m = orc.i128_to_int(orc.encode_i128(z, log_n, ls))
    assert m[0] == int(c * 2 ** ls) and abs(m[0]) > 1 << 63
    assert all(v == 0 for v in m[1:])


def test_wide_encode_decode_roundtrip_large_values(orc):
    rng = np.random.default_rng(7)
    z = rng.integers(0, 1 << 32, 1 << 14).astype(np.float64) + rng.uniform(-0.5, 0.5, 1 << 14)
    m = orc.encode_i128(z, 15, 55)
    assert max(abs(v) for v in orc.i128_to_int(m)) > 1 << 80
    assert np.max(np.abs(orc.decode_i128(m, 15, 55) - z)) < 1e-6


def test_wide_encryption_is_enc0_plus_m_and_decrypts(orc, P):
    """Eq. 4 literally: Enc(m) = Enc(0) + m with m's residues; the two-limb CRT of
    Dec recovers m + noise with |noise| <= 21 (2N + 1) (Theorem 1's bound, C-10)."""
    sk, sk_ntt, pk = orc.keygen(P, 3)
    rng = np.random.default_rng(8)
    m = [int(v) for v in rng.integers(-(1 << 62), 1 << 62, P.n)]
    m = [v * (1 << 30) + 17 for v in m]                     # |m| up to 2^92
    res = orc.residues_of_ints(P, m)
    for form in (0, 1):
        ct = orc.encrypt_general_explicit(P, pk, res, orc.sample_ternary(4, 0, 4, P.n),
                                          orc.sample_cbd(4, 0, 5, P.n), orc.sample_cbd(4, 0, 6, P.n), 1, form)
        zero = orc.vanilla_encrypt_explicit(P, pk, np.zeros(P.n, dtype=np.int64), orc.sample_ternary(4, 0, 4, P.n),
                                            orc.sample_cbd(4, 0, 5, P.n), orc.sample_cbd(4, 0, 6, P.n), form)
        # Enc(m) - Enc(0) = (m, 0) (in the form's domain)
        q = np.array([int(v) for v in P.q], dtype=object)[:, None]
        diff = ((ct[0].astype(object) - zero[0].astype(object)) % q).astype(np.uint64)
        want = res.copy()
        if form == 0:
            want = want.copy()
            from oracle import lib, _p, _u64p
            lib().orc_ntt_limbs(_p(want, _u64p), P.log_n, P.L, _p(P.q, _u64p), _p(P.psi, _u64p))
        assert np.array_equal(diff, want) and np.array_equal(ct[1], zero[1])
        x, st = orc.decrypt_wide(P, sk_ntt, ct, form)
        assert st == 0
        assert max(abs(a - b) for a, b in zip(x, m)) <= 21 * (2 * P.n + 1)


def test_two_limb_crt_equals_full_crt(orc, P):
    sk, sk_ntt, pk = orc.keygen(P, 5)
    m = [(1 << 100) - 12345 * j for j in range(P.n)]
    ct = orc.encrypt_general_explicit(P, pk, orc.residues_of_ints(P, m), orc.sample_ternary(6, 0, 4, P.n),
                                      orc.sample_cbd(6, 0, 5, P.n), orc.sample_cbd(6, 0, 6, P.n), 1, 1)
    x2, st = orc.decrypt_wide(P, sk_ntt, ct, 1)
    _, _, xl = orc.decrypt(P, sk_ntt, ct, 1, want_limbs=True)
    xf, _ = orc.crt_centered(P, xl)
    assert st == 0 and x2 == xf
