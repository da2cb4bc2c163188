"""Pins for the oracle's samplers (C-4): exact pmfs by chi-square, supports,
determinism, limb independence of the small samples, and the counter layout.

Statistical thresholds: chi-square at alpha = 1e-3, fixed seeds,
so the tests are deterministic.
"""
import math

import numpy as np
import pytest
from scipy import stats


def chi2_ok(observed, expected_p, alpha=1e-3):
    observed = np.asarray(observed, dtype=np.float64)
    exp = np.asarray(expected_p) * observed.sum()
    chi2 = float(((observed - exp) ** 2 / exp).sum())
    return stats.chi2.sf(chi2, len(observed) - 1) > alpha


def test_ternary_pmf(orc):
    x = orc.sample_ternary(1234, 7, orc.TAG_ENC_U, 1 << 17)
    assert set(np.unique(x).tolist()) <= {-1, 0, 1}
    counts = [(x == v).sum() for v in (-1, 0, 1)]
    assert chi2_ok(counts, [1 / 3] * 3)
    # frequencies within 3 sigma of 1/3
    n = len(x)
    for c in counts:
        assert abs(c / n - 1 / 3) < 3 * math.sqrt((1 / 3) * (2 / 3) / n)


def test_cbd_pmf(orc):
    x = orc.sample_cbd(99, 3, orc.TAG_ZINC_E1, 1 << 18)
    assert x.min() >= -21 and x.max() <= 21
    # exact pmf of Binomial(42, 1/2) - 21, tails pooled below expected count 5
    k = np.arange(-21, 22)
    p = stats.binom.pmf(k + 21, 42, 0.5)
    obs = np.array([(x == v).sum() for v in k])
    keep = p * len(x) >= 5
    obs_b = np.concatenate([obs[keep], [obs[~keep].sum()]])
    p_b = np.concatenate([p[keep], [p[~keep].sum()]])
    assert chi2_ok(obs_b, p_b)
    assert abs(x.mean()) < 4 * math.sqrt(10.5 / len(x))
    assert abs(x.var() - 10.5) / 10.5 < 0.02


def test_uniform_mod_q(orc):
    q = 18014398508400641
    x = orc.sample_uniform(5, 0, orc.TAG_PK_A, 3, q, 1 << 16).astype(np.float64)
    assert (x < q).all()
    buckets = np.floor(x / q * 16).astype(int)
    assert chi2_ok(np.bincount(buckets, minlength=16), [1 / 16] * 16)


def test_determinism_and_stream_separation(orc):
    a = orc.sample_cbd(1, 2, orc.TAG_ENC_E1, 4096)
    assert np.array_equal(a, orc.sample_cbd(1, 2, orc.TAG_ENC_E1, 4096))
    assert not np.array_equal(a, orc.sample_cbd(1, 2, orc.TAG_ENC_E2, 4096))
    assert not np.array_equal(a, orc.sample_cbd(1, 3, orc.TAG_ENC_E1, 4096))
    assert not np.array_equal(a, orc.sample_cbd(2, 2, orc.TAG_ENC_E1, 4096))
    # a prefix of a longer draw is the shorter draw (counter = coefficient block)
    assert np.array_equal(orc.sample_cbd(1, 2, orc.TAG_ENC_E1, 8192)[:4096], a)
    # message indices above 2^32 use the high counter word
    assert not np.array_equal(orc.sample_cbd(1, 2 + (1 << 32), orc.TAG_ENC_E1, 4096), a)


def test_counter_layout(orc):
    """C-4 layout: counter (block, msg_lo, msg_hi, tag<<16|limb), key (seed_lo, seed_hi).
    (This documents the convention both implementations follow.)"""
    seed, msg = 0x0123456789ABCDEF, 0xFEDCBA9876543210
    key = [seed & 0xFFFFFFFF, seed >> 32]
    t = orc.sample_ternary(seed, msg, orc.TAG_ENC_U, 8)
    c = orc.sample_cbd(seed, msg, orc.TAG_ZINC_E2, 4)
    for blk in range(2):
        w = orc.philox4x32_10([blk, msg & 0xFFFFFFFF, msg >> 32, orc.TAG_ENC_U << 16], key)
        for r in range(4):
            assert t[4 * blk + r] == ((int(w[r]) * 3) >> 32) - 1
    for blk in range(2):
        w = [int(v) for v in orc.philox4x32_10([blk, msg & 0xFFFFFFFF, msg >> 32, orc.TAG_ZINC_E2 << 16], key)]
        m = (1 << 21) - 1
        for r in range(2):
            assert c[2 * blk + r] == bin(w[2 * r] & m).count("1") - bin(w[2 * r + 1] & m).count("1")
    q = 68719403009
    u = orc.sample_uniform(seed, 0, orc.TAG_PK_A, 2, q, 3)
    for blk in range(3):
        w = [int(v) for v in orc.philox4x32_10([blk, 0, 0, (orc.TAG_PK_A << 16) | 2], key)]
        assert int(u[blk]) == (w[0] | w[1] << 32 | w[2] << 64 | w[3] << 96) % q
