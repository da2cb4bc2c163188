"""GPU parity of the wide-plaintext path: the paper's own
parameters, N = 2^15, 15 x 55-bit + one 56-bit prime (881-bit Q), Delta = 2^55
(PAPER.md:349-351).  128-bit integer plaintexts give ciphertexts bit-exact with the
oracle (Enc(0) + m, Eq. 4); wide decryption recovers x by a two-limb CRT exactly as
the oracle's big-integer one; slot values of the paper's dataset ranges (hg38 "less
than 2^9"; Bitcoin-like up to 2^32) round-trip within tolerance."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

NTT, COEFF = 0, 1
BITS = [56] + [55] * 15


@pytest.fixture(scope="module")
def Z():
    import paper_2408_07304_b200 as Z
    return Z


@pytest.fixture(scope="module")
def S(Z, orc):
    ctx = Z.Context(15, BITS, 55)
    P = orc.Params.make(15, BITS, 55)
    sk, _, pk = Z.zinc_keygen(ctx, 201)
    o_sk, o_sk_ntt, o_pk = orc.keygen(P, 201)
    caches = {f: Z.zinc_precompute_cache(ctx, pk, 202, f) for f in (NTT, COEFF)}
    return ctx, P, sk, pk, o_sk_ntt, o_pk, caches


def add_residues(orc, P, ct, ints, form):
    res = orc.residues_of_ints(P, ints)
    if form == NTT:
        res = orc.ntt_limbs(P, res)
    q = np.array([int(v) for v in P.q], dtype=object)[:, None]
    out = ct.copy()
    out[0] = ((ct[0].astype(object) + res.astype(object)) % q).astype(np.uint64)
    return out


@pytest.mark.parametrize("path", ["zinc", "vanilla"])
@pytest.mark.parametrize("form", [NTT, COEFF])
def test_i128_plaintexts_bit_exact_and_wide_decrypt(Z, orc, S, path, form):
    ctx, P, sk, pk, o_sk_ntt, o_pk, caches = S
    B = 3
    rng = np.random.default_rng([7, form, len(path)])
    ints = [[int(v) * (1 << 40) + int(w) for v, w in zip(rng.integers(-(1 << 60), 1 << 60, P.n),
                                                        rng.integers(0, 1 << 40, P.n))] for _ in range(B)]
    m = torch.from_numpy(np.stack([orc.int_to_i128(v) for v in ints])).cuda()
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(ctx, caches[form], form, m, 11, 500)
        o_cache = orc.precompute_cache(P, o_pk, 202, form)
    else:
        ct = Z.ckks_encrypt_batch(ctx, pk, form, m, 11, 500)
    got = ct.cpu().numpy()
    zero = np.zeros(P.n, dtype=np.int64)
    for b in (0, B - 1):
        base = (orc.zinc_encrypt(P, o_cache, form, zero, 11, 500 + b) if path == "zinc"
                else orc.vanilla_encrypt(P, o_pk, zero, 11, 500 + b, form))
        assert np.array_equal(got[b], add_residues(orc, P, base, ints[b], form)), b
    x, status, _ = Z.ckks_decrypt_batch_wide(ctx, sk, form, ct, slots=False)
    assert (status.cpu().numpy() == 0).all()
    xs = orc.i128_to_int(x[1].cpu().numpy())
    want, st = orc.decrypt_wide(P, o_sk_ntt, got[1], form)
    assert st == 0 and xs == want
    assert max(abs(a - b) for a, b in zip(xs, ints[1])) <= 21 * (3 * P.n + 2)


@pytest.mark.parametrize("shape", ["hg38", "bitcoin"])
def test_paper_value_ranges_from_slots(Z, orc, S, shape):
    """Stand-ins with the paper's value ranges (DESIGN.md f3): GPU wide encode within
    2^-45 (relative) of the oracle's long-double encode; the slot path equals the
    I128 path on the GPU's own encoding; decode within 1e-4."""
    ctx, P, sk, pk, o_sk_ntt, o_pk, caches = S
    rng = np.random.default_rng(3)
    M = P.n // 2
    z = np.zeros((4, M))
    if shape == "hg38":  # every slot a value below 2^9: m_0 = Delta mean(z) reaches ~2^63
        z[:] = rng.integers(0, 1 << 9, (4, M))
    else:
        z[:, 0] = rng.integers(1 << 20, 1 << 32, 4)
        z[:, 1:M:97] = rng.uniform(-1 << 31, 1 << 31, (4, len(range(1, M, 97))))
    zd = torch.from_numpy(z).cuda()
    m = Z.ckks_encode_batch_wide(ctx, zd)
    mi = orc.i128_to_int(m[0].cpu().numpy())
    oi = orc.i128_to_int(orc.encode_i128(z[0], 15, 55))
    scale = max(abs(v) for v in oi)
    assert scale > 1 << 62
    assert max(abs(a - b) for a, b in zip(mi, oi)) <= scale / 2 ** 45
    for form in (COEFF, NTT):
        a = Z.zinc_encrypt_batch(ctx, caches[form], form, zd, 5, 0)
        b = Z.zinc_encrypt_batch(ctx, caches[form], form, m, 5, 0)
        assert torch.equal(a, b)
        _, st, zz = Z.ckks_decrypt_batch(ctx, sk, form, a)
        assert (st.cpu().numpy() == 0).all()
        assert np.max(np.abs(zz.cpu().numpy() - z)) < 1e-4


def test_i128_tiny_high_word_edges_bit_exact(Z, orc, S):
    """The add/inject kernel's "tiny high word" path (|hi| < 2^7 at 56-bit primes, decided per warp
    after e1' is added with its carry into hi): plaintexts at its boundaries -- hi in {0, +-1, +-126,
    +-127, +-128, 129}, lo in {0, 1, 20, 2^63, 2^64 - 21, 2^64 - 1} (so that e1' carries or borrows
    across 2^64), one message all tiny, one with a non-tiny coefficient in every warp, one mixing
    warps -- bit-exact against Enc(0) + residues of the integers (Eq. 4)."""
    ctx, P, sk, pk, o_sk_ntt, o_pk, caches = S
    his = [0, 1, -1, 126, -126, 127, -127, 2, -2, 64]
    his_edge = [128, -128, 129, -129, 127, -127, 0, 1000, -(1 << 40)]
    los = [0, 1, 20, 1 << 63, (1 << 64) - 21, (1 << 64) - 1, 12345678901234567, (1 << 64) - 5]
    rng = np.random.default_rng(77)

    def msg(kind):
        out = []
        for j in range(P.n):
            hi = his[rng.integers(len(his))]
            if kind == 1 and j % 64 == 17:
                hi = his_edge[rng.integers(len(his_edge))]
            if kind == 2 and (j // 64) % 3 == 0:
                hi = his_edge[rng.integers(len(his_edge))]
            out.append(hi * (1 << 64) + los[rng.integers(len(los))])
        return out

    ints = [msg(k) for k in (0, 1, 2)]
    m = torch.from_numpy(np.stack([orc.int_to_i128(v) for v in ints])).cuda()
    ct = Z.zinc_encrypt_batch(ctx, caches[COEFF], COEFF, m, 13, 900).cpu().numpy()
    o_cache = orc.precompute_cache(P, o_pk, 202, COEFF)
    zero = np.zeros(P.n, dtype=np.int64)
    for b in range(3):
        base = orc.zinc_encrypt(P, o_cache, COEFF, zero, 13, 900 + b)
        assert np.array_equal(ct[b], add_residues(orc, P, base, ints[b], COEFF)), b
