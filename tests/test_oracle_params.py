"""Pins for the oracle's parameter generation (C-1 primes, C-2 psi) and Philox (C-4).

Each check uses something other than the oracle itself: Python big-int
arithmetic (``pow``), exhaustive scans, trial division, the SURVEY Appendix A
values (computed by an independent script), and the Random123 known-answer
vectors for Philox4x32-10.
"""
import json
import math
import os
import random

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def py_is_prime(n: int) -> bool:
    """Independent Miller-Rabin in Python big ints: 40 random bases + fixed ones."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47]
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    rng = random.Random(n)
    for a in small + [rng.randrange(2, n - 1) for _ in range(40)]:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def trial_division_is_prime(n: int) -> bool:
    if n < 2:
        return False
    i = 2
    while i * i <= n:
        if n % i == 0:
            return False
        i += 1
    return True


def test_is_prime_matches_trial_division(orc):
    for n in list(range(0, 3000)) + [561, 1105, 1729, 2465, 2821, 6601, 8911, 41041, 825265]:
        assert orc.is_prime(n) == trial_division_is_prime(n), n
    # strong pseudoprimes to many small bases (fool weak MR variants)
    for n in [3215031751, 2152302898747, 3474749660383, 341550071728321, 3825123056546413051]:
        assert not orc.is_prime(n), n
    # known primes
    for n in [2**61 - 1, 2**31 - 1, 1000000007, 998244353]:
        assert orc.is_prime(n)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_primes_and_psi_appendix_a(orc, name):
    g = json.load(open(os.path.join(GOLD, "params_appendix_a.json")))[name]
    P = orc.Params.make(g["log_n"], g["bits"], 40)
    assert [int(x) for x in P.q] == g["q"]
    assert [int(x) for x in P.psi] == g["psi"]
    log_q = sum(math.log2(int(x)) for x in P.q)
    assert abs(log_q - g["log_q"]) < 0.01


@pytest.mark.parametrize("log_n,bits", [(12, [36] * 3), (13, [60, 40, 40, 60]), (14, [54] * 8), (10, [30, 30, 45])])
def test_primes_are_the_largest(orc, log_n, bits):
    """C-1 from its definition: prime, = 1 mod 2N, < 2^b, and no unused prime
    candidate of that form lies above it (checked with Python big ints)."""
    q = [int(x) for x in orc.find_primes(log_n, bits)]
    two_n = 2 << log_n
    for i, (qi, b) in enumerate(zip(q, bits)):
        assert py_is_prime(qi)
        assert qi % two_n == 1
        assert qi < 2**b and qi.bit_length() == b
        taken = {q[j] for j in range(i) if bits[j] == b}
        c = qi + two_n
        while c < 2**b:
            assert c in taken or not py_is_prime(c), (qi, c)
            c += two_n
    # repeated sizes descend
    for b in set(bits):
        same = [qi for qi, bb in zip(q, bits) if bb == b]
        assert same == sorted(same, reverse=True) and len(set(same)) == len(same)


@pytest.mark.parametrize("log_n,bits", [(12, [36] * 3), (13, [60, 40, 40, 60]), (14, [54] * 8)])
def test_psi_is_smallest_primitive_root(orc, log_n, bits):
    """C-2 from its definition: psi^N = -1 (so psi has order exactly 2N), and psi
    is the minimum over all primitive 2N-th roots = {psi^k : k odd} (scan)."""
    n = 1 << log_n
    P = orc.Params.make(log_n, bits, 40)
    for qi, psi in zip(map(int, P.q), map(int, P.psi)):
        assert pow(psi, n, qi) == qi - 1
        assert pow(psi, 2 * n, qi) == 1
        p2 = psi * psi % qi
        x, best = psi, psi
        for _ in range(n):
            best = min(best, x)
            x = x * p2 % qi
        assert best == psi


def test_philox_known_answer_vectors(orc):
    path = os.path.join(GOLD, "philox4x32_10_kat.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = orc.philox4x32_10(v[0:4], v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_philox_counter_sensitivity(orc):
    base = orc.philox4x32_10([1, 2, 3, 4], [5, 6])
    for i in range(4):
        c = [1, 2, 3, 4]
        c[i] ^= 1
        assert not np.array_equal(orc.philox4x32_10(c, [5, 6]), base)
    assert not np.array_equal(orc.philox4x32_10([1, 2, 3, 4], [5, 7]), base)
