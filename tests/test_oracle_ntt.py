"""Pins for the oracle's negacyclic NTT (C-3) and schoolbook product.

Independent checks: evaluation of a(X) at psi^(2 brv(k) + 1) by Horner in
Python big ints; the convolution theorem against a Python/numpy schoolbook
negacyclic product; the X^i X^j sign rule; constant polynomials
(SPEC.md:70); inverse round trip.
"""
import numpy as np
import pytest

Q36 = 68719403009   # C1 limb 0 (N = 4096 -> valid for log_n <= 12)


def brv(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def params_for(orc, log_n, b=36):
    q = int(orc.find_primes(log_n, [b])[0])
    return q, orc.min_psi(q, log_n)


def py_eval_ntt(a, log_n, q, psi, ks):
    out = []
    for k in ks:
        r = pow(psi, 2 * brv(k, log_n) + 1, q)
        acc = 0
        for c in reversed([int(x) for x in a]):
            acc = (acc * r + c) % q
        out.append(acc)
    return out


def py_negacyclic(a, b, q):
    n = len(a)
    out = [0] * n
    for i in range(n):
        ai = int(a[i])
        if ai == 0:
            continue
        for j in range(n):
            p = ai * int(b[j])
            if i + j < n:
                out[i + j] += p
            else:
                out[i + j - n] -= p
    return [x % q for x in out]


@pytest.mark.parametrize("log_n", [1, 2, 3, 4, 5, 6])
def test_ntt_definition_is_evaluation_at_odd_powers(orc, log_n):
    n = 1 << log_n
    q, psi = params_for(orc, log_n, 40)
    rng = np.random.default_rng(log_n)
    a = rng.integers(0, q, n, dtype=np.uint64)
    assert [int(x) for x in orc.ntt_definition(a, log_n, q, psi)] == py_eval_ntt(a, log_n, q, psi, range(n))
    assert [int(x) for x in orc.ntt(a, log_n, q, psi)] == py_eval_ntt(a, log_n, q, psi, range(n))


@pytest.mark.parametrize("log_n", [7, 8, 10])
def test_iterative_ntt_equals_definition(orc, log_n):
    q, psi = params_for(orc, log_n, 54)
    rng = np.random.default_rng(100 + log_n)
    a = rng.integers(0, q, 1 << log_n, dtype=np.uint64)
    assert np.array_equal(orc.ntt(a, log_n, q, psi), orc.ntt_definition(a, log_n, q, psi))


@pytest.mark.parametrize("log_n,b", [(12, 36), (13, 60), (14, 54), (15, 55)])
def test_full_size_spot_coefficients_and_roundtrip(orc, log_n, b):
    q, psi = params_for(orc, log_n, b)
    rng = np.random.default_rng(log_n)
    a = rng.integers(0, q, 1 << log_n, dtype=np.uint64)
    A = orc.ntt(a, log_n, q, psi)
    ks = [0, 1, 2, (1 << log_n) - 1, 12345 % (1 << log_n)]
    assert [int(A[k]) for k in ks] == py_eval_ntt(a, log_n, q, psi, ks)
    assert np.array_equal(orc.intt(A, log_n, q, psi), a)


@pytest.mark.parametrize("log_n", [4, 5, 6, 8])
def test_convolution_theorem_vs_python_schoolbook(orc, log_n):
    q, psi = params_for(orc, log_n, 50)
    rng = np.random.default_rng(7 * log_n)
    for _ in range(3):
        a = rng.integers(0, q, 1 << log_n, dtype=np.uint64)
        b = rng.integers(0, q, 1 << log_n, dtype=np.uint64)
        A, B = orc.ntt(a, log_n, q, psi), orc.ntt(b, log_n, q, psi)
        C = np.array([int(x) * int(y) % q for x, y in zip(A, B)], dtype=np.uint64)
        expect = py_negacyclic(a, b, q)
        assert [int(x) for x in orc.intt(C, log_n, q, psi)] == expect
        assert [int(x) for x in orc.polymul_schoolbook(a, b, log_n, q)] == expect


def test_negacyclic_sign_rule_exhaustive_n8(orc):
    """X^i X^j = sign X^((i+j) mod N), sign = -1 iff i + j >= N."""
    log_n, n = 3, 8
    q, psi = params_for(orc, log_n, 30)
    for i in range(n):
        for j in range(n):
            a = np.zeros(n, dtype=np.uint64); a[i] = 1
            b = np.zeros(n, dtype=np.uint64); b[j] = 1
            A, B = orc.ntt(a, log_n, q, psi), orc.ntt(b, log_n, q, psi)
            C = np.array([int(x) * int(y) % q for x, y in zip(A, B)], dtype=np.uint64)
            c = orc.intt(C, log_n, q, psi)
            e = np.zeros(n, dtype=np.uint64)
            e[(i + j) % n] = 1 if i + j < n else q - 1
            assert np.array_equal(c, e), (i, j)


def test_constant_polynomial_maps_to_constant_vector(orc):
    """SPEC.md:70."""
    log_n = 12
    q, psi = params_for(orc, log_n, 36)
    a = np.zeros(1 << log_n, dtype=np.uint64)
    a[0] = 123456789
    assert (orc.ntt(a, log_n, q, psi) == 123456789).all()


def test_transform_counter(orc):
    q, psi = params_for(orc, 6, 36)
    orc.counters_reset()
    a = np.arange(64, dtype=np.uint64)
    orc.intt(orc.ntt(a, 6, q, psi), 6, q, psi)
    assert orc.counters()[0] == 2
