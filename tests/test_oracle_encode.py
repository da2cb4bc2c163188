"""Pins for the oracle's CKKS encoding / decoding (C-6, C-10 decode).

Independent checks: the two closed forms, the defining
property of the canonical embedding m(zeta^(5^k)) = Delta z_k evaluated with
numpy's FFT (a library routine), the O(N log N) encoder against the O(N^2)
definition, and decode(encode(z)) within the rounding bound.
"""
import math

import numpy as np
import pytest


def eval_at_5k_roots(m, log_n):
    """m(zeta^(g_k)), g_k = 5^k mod 2N, zeta = exp(i pi / N), via numpy FFT:
    m(zeta^(2l+1)) = sum_j (m_j zeta^j) exp(2 pi i l j / N) = N * ifft(m zeta^j)[l]."""
    n = 1 << log_n
    j = np.arange(n)
    vals = np.fft.ifft(np.asarray(m, dtype=np.float64) * np.exp(1j * np.pi * j / n)) * n
    g = 1
    out = np.empty(n // 2, dtype=np.complex128)
    for k in range(n // 2):
        out[k] = vals[(g - 1) // 2]
        g = g * 5 % (2 * n)
    return out


def near_half(x):
    return abs((x - math.floor(x)) - 0.5) < 1e-6


@pytest.mark.parametrize("log_n,log_scale", [(3, 20), (6, 30), (10, 40), (12, 30)])
def test_closed_form_constant_slots(orc, log_n, log_scale):
    c = 0.3718281828
    z = np.full(1 << (log_n - 1), c)
    for enc in (orc.encode_definition, orc.encode):
        m = enc(z, log_n, log_scale)
        assert m[0] == round(c * 2.0 ** log_scale)
        assert (m[1:] == 0).all()


@pytest.mark.parametrize("log_n,log_scale", [(3, 20), (8, 30), (12, 40)])
def test_closed_form_unit_slot(orc, log_n, log_scale):
    n = 1 << log_n
    z = np.zeros(n // 2)
    z[0] = 1.0
    for enc in (orc.encode_definition, orc.encode):
        m = enc(z, log_n, log_scale)
        for j in range(n):
            x = (2.0 ** (log_scale + 1) / n) * math.cos(math.pi * j / n)
            if near_half(x):
                assert abs(m[j] - x) <= 1
            else:
                assert m[j] == int(math.floor(abs(x) + 0.5)) * (1 if x >= 0 else -1), j


@pytest.mark.parametrize("log_n,log_scale,cplx", [(4, 20, False), (9, 30, True), (12, 30, False), (14, 40, False)])
def test_canonical_embedding_property(orc, log_n, log_scale, cplx):
    """m(zeta^(5^k)) = Delta z_k up to the rounding of m (|err| <= N/2 / Delta)."""
    n = 1 << log_n
    rng = np.random.default_rng(log_n)
    z = rng.uniform(-1, 1, n // 2) + (1j * rng.uniform(-1, 1, n // 2) if cplx else 0)
    m = orc.encode(z, log_n, log_scale)
    got = eval_at_5k_roots(m, log_n) / 2.0 ** log_scale
    assert np.max(np.abs(got - z)) <= (n / 2) / 2.0 ** log_scale
    # and decode, which is that evaluation by definition
    assert np.max(np.abs(orc.decode(m, log_n, log_scale) - got)) < 1e-9


@pytest.mark.parametrize("log_n,log_scale,cplx", [(3, 20, True), (7, 30, False), (10, 40, True), (12, 30, False)])
def test_fft_encode_equals_definition(orc, log_n, log_scale, cplx):
    n = 1 << log_n
    rng = np.random.default_rng(1000 + log_n)
    z = rng.uniform(-1, 1, n // 2) + (1j * rng.uniform(-1, 1, n // 2) if cplx else 0)
    a = orc.encode_definition(z, log_n, log_scale)
    b = orc.encode(z, log_n, log_scale)
    assert np.max(np.abs(a - b)) <= 1
    assert np.mean(a == b) > 0.999


def test_fft_encode_equals_definition_full_c3(orc):
    """Full C3 size (N = 2^14, Delta = 2^40): the O(N^2) definition vs the FFT form."""
    log_n, log_scale = 14, 40
    rng = np.random.default_rng(3)
    z = np.clip(rng.standard_normal(1 << 13), -4, 4)
    a = orc.encode_definition(z, log_n, log_scale)
    b = orc.encode(z, log_n, log_scale)
    assert np.max(np.abs(a - b)) <= 1


@pytest.mark.parametrize("log_n,log_scale", [(6, 30), (10, 30), (12, 40)])
def test_decode_definition_equals_fft_and_roundtrip(orc, log_n, log_scale):
    n = 1 << log_n
    rng = np.random.default_rng(log_n + 7)
    z = rng.uniform(-1, 1, n // 2) + 1j * rng.uniform(-1, 1, n // 2)
    m = orc.encode(z, log_n, log_scale)
    d1 = orc.decode_definition(m, log_n, log_scale)
    d2 = orc.decode(m, log_n, log_scale)
    assert np.max(np.abs(d1 - d2)) < 1e-9
    # rounding bound: each coefficient moves by <= 1/2, so |err| <= N/(2 Delta)
    assert np.max(np.abs(d2 - z)) <= n / 2 / 2.0 ** log_scale
