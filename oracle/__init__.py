"""CPU oracle for the Zinc hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around ``oracle/oracle.c`` (plain C, ``unsigned __int128``
with ``%``, long double encoding).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It never imports ``paper_2408_07304_b200`` and the CUDA library never
imports it.  Conventions C-1..C-10: ``docs/CONVENTIONS.md``.

Layouts (numpy, C order): polynomial ``[N]``; RNS polynomial ``[L][N]`` uint64
canonical residues; ciphertext / public key / cache ``[2][L][N]`` uint64 with
component 0 = the paper's c1 (carries m) and 1 = c2.
Forms: ``NTT = 0``, ``COEFF = 1`` (reading A4).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NTT, COEFF = 0, 1
TAG_SK, TAG_PK_E, TAG_PK_A, TAG_ENC_U, TAG_ENC_E1, TAG_ENC_E2, TAG_ZINC_E1, TAG_ZINC_E2 = range(1, 9)
CACHE_MSG = (1 << 64) - 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_c = ctypes


def _declare(L):
    sig = {
        "orc_counters_reset": (None, []),
        "orc_counters_get": (None, [_u64p, _u64p]),
        "orc_is_prime": (_c.c_int, [_c.c_uint64]),
        "orc_find_primes": (_c.c_int, [_c.c_int, _c.c_int, _i32p, _u64p]),
        "orc_min_psi": (_c.c_uint64, [_c.c_uint64, _c.c_int]),
        "orc_philox4x32_10": (None, [_u32p, _u32p, _u32p]),
        "orc_sample_ternary": (None, [_c.c_uint64, _c.c_uint64, _c.c_uint32, _c.c_int, _i64p]),
        "orc_sample_cbd": (None, [_c.c_uint64, _c.c_uint64, _c.c_uint32, _c.c_int, _i64p]),
        "orc_sample_uniform": (None, [_c.c_uint64, _c.c_uint64, _c.c_uint32, _c.c_uint32, _c.c_uint64, _c.c_int, _u64p]),
        "orc_ntt_definition": (None, [_u64p, _c.c_int, _c.c_uint64, _c.c_uint64, _u64p]),
        "orc_ntt": (None, [_u64p, _c.c_int, _c.c_uint64, _c.c_uint64]),
        "orc_intt": (None, [_u64p, _c.c_int, _c.c_uint64, _c.c_uint64]),
        "orc_polymul_schoolbook": (None, [_u64p, _u64p, _c.c_int, _c.c_uint64, _u64p]),
        "orc_encode_definition": (None, [_f64p, _f64p, _c.c_int, _c.c_int, _i64p]),
        "orc_encode_fft": (None, [_f64p, _f64p, _c.c_int, _c.c_int, _i64p]),
        "orc_decode_definition": (None, [_i64p, _c.c_int, _c.c_int, _f64p, _f64p]),
        "orc_decode_fft": (None, [_i64p, _c.c_int, _c.c_int, _f64p, _f64p]),
        "orc_keygen": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _c.c_uint64, _i64p, _u64p, _u64p]),
        "orc_vanilla_encrypt_explicit": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _i64p, _i64p, _i64p, _i64p, _c.c_int, _u64p]),
        "orc_vanilla_encrypt": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _i64p, _c.c_uint64, _c.c_uint64, _c.c_int, _u64p]),
        "orc_precompute_cache": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _c.c_uint64, _c.c_int, _u64p]),
        "orc_zinc_encrypt_explicit": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _c.c_int, _i64p, _i64p, _i64p, _u64p]),
        "orc_zinc_encrypt": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _c.c_int, _i64p, _c.c_uint64, _c.c_uint64, _u64p]),
        "orc_decrypt": (_c.c_int, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _u64p, _c.c_int, _i64p, _u64p]),
        "orc_ntt_limbs": (None, [_u64p, _c.c_int, _c.c_int, _u64p, _u64p]),
        "orc_encode_fft_i128": (None, [_f64p, _f64p, _c.c_int, _c.c_int, _i64p]),
        "orc_decode_fft_i128": (None, [_i64p, _c.c_int, _c.c_int, _f64p, _f64p]),
        "orc_ct_add": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _c.c_uint64, _u64p]),
        "orc_ct_sum": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _c.c_uint64, _u64p]),
        "orc_keygen_scaled": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _c.c_uint64, _c.c_int64, _i64p, _u64p, _u64p]),
        "orc_bfv_delta_mod": (_c.c_uint64, [_c.c_int, _u64p, _c.c_uint64, _c.c_int]),
        "orc_plaintext_residues": (None, [_c.c_int, _c.c_uint64, _c.c_int, _c.c_int, _u64p, _i64p, _u64p]),
        "orc_encrypt_general_explicit": (None, [_c.c_int, _c.c_int, _u64p, _u64p, _u64p, _u64p, _i64p, _i64p, _i64p, _c.c_int64, _c.c_int, _u64p]),
        "orc_encrypt_scheme": (None, [_c.c_int, _c.c_uint64, _c.c_int, _c.c_int, _u64p, _u64p, _u64p, _i64p, _c.c_uint64, _c.c_uint64, _c.c_int, _u64p]),
        "orc_precompute_cache_scheme": (None, [_c.c_int, _c.c_uint64, _c.c_int, _c.c_int, _u64p, _u64p, _u64p, _c.c_uint64, _c.c_int, _u64p]),
        "orc_zinc_encrypt_scheme": (None, [_c.c_int, _c.c_uint64, _c.c_int, _c.c_int, _u64p, _u64p, _u64p, _c.c_int, _i64p, _c.c_uint64, _c.c_uint64, _u64p]),
        "orc_intt_limbs": (None, [_u64p, _c.c_int, _c.c_int, _u64p, _u64p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _p(a: np.ndarray, ptype):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ptype)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------- parameters
def is_prime(n: int) -> bool:
    return bool(lib().orc_is_prime(n))


def find_primes(log_n: int, bits) -> np.ndarray:
    bits_a = np.ascontiguousarray(bits, dtype=np.int32)
    q = np.zeros(len(bits_a), dtype=np.uint64)
    rc = lib().orc_find_primes(log_n, len(bits_a), _p(bits_a, _i32p), _p(q, _u64p))
    if rc != 0:
        raise ValueError("no prime found")
    return q


def min_psi(q: int, log_n: int) -> int:
    return int(lib().orc_min_psi(int(q), log_n))


@dataclass
class Params:
    """Ring/RNS parameters per C-1, C-2."""
    log_n: int
    bits: tuple
    log_scale: int
    q: np.ndarray
    psi: np.ndarray

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def L(self) -> int:
        return len(self.bits)

    @classmethod
    def make(cls, log_n: int, bits, log_scale: int) -> "Params":
        q = find_primes(log_n, bits)
        psi = np.array([min_psi(int(qi), log_n) for qi in q], dtype=np.uint64)
        return cls(log_n, tuple(int(b) for b in bits), log_scale, q, psi)

    def _args(self):
        return self.log_n, self.L, _p(self.q, _u64p), _p(self.psi, _u64p)


# ---------------------------------------------------------------- randomness
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c, _u32p), _p(k, _u32p), _p(out, _u32p))
    return out


def sample_ternary(seed: int, msg: int, tag: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.int64)
    lib().orc_sample_ternary(seed, msg, tag, n, _p(out, _i64p))
    return out


def sample_cbd(seed: int, msg: int, tag: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.int64)
    lib().orc_sample_cbd(seed, msg, tag, n, _p(out, _i64p))
    return out


def sample_uniform(seed: int, msg: int, tag: int, limb: int, q: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().orc_sample_uniform(seed, msg, tag, limb, int(q), n, _p(out, _u64p))
    return out


# ---------------------------------------------------------------- transforms
def ntt_definition(a, log_n: int, q: int, psi: int) -> np.ndarray:
    a = _u64(a)
    out = np.zeros_like(a)
    lib().orc_ntt_definition(_p(a, _u64p), log_n, int(q), int(psi), _p(out, _u64p))
    return out


def ntt(a, log_n: int, q: int, psi: int) -> np.ndarray:
    a = _u64(a).copy()
    lib().orc_ntt(_p(a, _u64p), log_n, int(q), int(psi))
    return a


def intt(a, log_n: int, q: int, psi: int) -> np.ndarray:
    a = _u64(a).copy()
    lib().orc_intt(_p(a, _u64p), log_n, int(q), int(psi))
    return a


def ntt_limbs(P: Params, a) -> np.ndarray:
    a = _u64(a).copy()
    lib().orc_ntt_limbs(_p(a, _u64p), P.log_n, P.L, _p(P.q, _u64p), _p(P.psi, _u64p))
    return a


def intt_limbs(P: Params, a) -> np.ndarray:
    a = _u64(a).copy()
    lib().orc_intt_limbs(_p(a, _u64p), P.log_n, P.L, _p(P.q, _u64p), _p(P.psi, _u64p))
    return a


def polymul_schoolbook(a, b, log_n: int, q: int) -> np.ndarray:
    a, b = _u64(a), _u64(b)
    out = np.zeros_like(a)
    lib().orc_polymul_schoolbook(_p(a, _u64p), _p(b, _u64p), log_n, int(q), _p(out, _u64p))
    return out


# ---------------------------------------------------------------- encoding
def _slots(z):
    z = np.asarray(z)
    re = np.ascontiguousarray(z.real, dtype=np.float64)
    im = np.ascontiguousarray(z.imag if np.iscomplexobj(z) else np.zeros_like(re), dtype=np.float64)
    return re, im


def encode_definition(z, log_n: int, log_scale: int) -> np.ndarray:
    re, im = _slots(z)
    m = np.zeros(1 << log_n, dtype=np.int64)
    lib().orc_encode_definition(_p(re, _f64p), _p(im, _f64p), log_n, log_scale, _p(m, _i64p))
    return m


def encode(z, log_n: int, log_scale: int) -> np.ndarray:
    """O(N log N) encode (pinned to encode_definition)."""
    re, im = _slots(z)
    m = np.zeros(1 << log_n, dtype=np.int64)
    lib().orc_encode_fft(_p(re, _f64p), _p(im, _f64p), log_n, log_scale, _p(m, _i64p))
    return m


def decode_definition(x, log_n: int, log_scale: int) -> np.ndarray:
    x = _i64(x)
    re = np.zeros(1 << (log_n - 1)); im = np.zeros_like(re)
    lib().orc_decode_definition(_p(x, _i64p), log_n, log_scale, _p(re, _f64p), _p(im, _f64p))
    return re + 1j * im


def decode(x, log_n: int, log_scale: int) -> np.ndarray:
    x = _i64(x)
    re = np.zeros(1 << (log_n - 1)); im = np.zeros_like(re)
    lib().orc_decode_fft(_p(x, _i64p), log_n, log_scale, _p(re, _f64p), _p(im, _f64p))
    return re + 1j * im


# ---------------------------------------------------------------- scheme
def keygen(P: Params, seed: int):
    """Returns (sk_coeff int64[N], sk_ntt uint64[L][N], pk_ntt uint64[2][L][N])."""
    sk = np.zeros(P.n, dtype=np.int64)
    sk_ntt = np.zeros((P.L, P.n), dtype=np.uint64)
    pk = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_keygen(*P._args(), seed, _p(sk, _i64p), _p(sk_ntt, _u64p), _p(pk, _u64p))
    return sk, sk_ntt, pk


def vanilla_encrypt_explicit(P: Params, pk, m, u, e1, e2, form: int) -> np.ndarray:
    pk, m, u, e1, e2 = _u64(pk), _i64(m), _i64(u), _i64(e1), _i64(e2)
    ct = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_vanilla_encrypt_explicit(*P._args(), _p(pk, _u64p), _p(m, _i64p), _p(u, _i64p),
                                       _p(e1, _i64p), _p(e2, _i64p), form, _p(ct, _u64p))
    return ct


def vanilla_encrypt(P: Params, pk, m, seed: int, msg: int, form: int) -> np.ndarray:
    pk, m = _u64(pk), _i64(m)
    ct = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_vanilla_encrypt(*P._args(), _p(pk, _u64p), _p(m, _i64p), seed, msg, form, _p(ct, _u64p))
    return ct


def precompute_cache(P: Params, pk, cache_seed: int, form: int) -> np.ndarray:
    pk = _u64(pk)
    cache = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_precompute_cache(*P._args(), _p(pk, _u64p), cache_seed, form, _p(cache, _u64p))
    return cache


def zinc_encrypt_explicit(P: Params, cache, form: int, m, e1p, e2p) -> np.ndarray:
    cache, m, e1p, e2p = _u64(cache), _i64(m), _i64(e1p), _i64(e2p)
    ct = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_zinc_encrypt_explicit(*P._args(), _p(cache, _u64p), form, _p(m, _i64p),
                                    _p(e1p, _i64p), _p(e2p, _i64p), _p(ct, _u64p))
    return ct


def zinc_encrypt(P: Params, cache, form: int, m, seed: int, msg: int) -> np.ndarray:
    cache, m = _u64(cache), _i64(m)
    ct = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_zinc_encrypt(*P._args(), _p(cache, _u64p), form, _p(m, _i64p), seed, msg, _p(ct, _u64p))
    return ct


def decrypt(P: Params, sk_ntt, ct, form: int, want_limbs: bool = False):
    """Returns (x centered mod q0 int64[N], status 0/1[, x_limbs [L][N]])."""
    sk_ntt, ct = _u64(sk_ntt), _u64(ct)
    x = np.zeros(P.n, dtype=np.int64)
    xl = np.zeros((P.L, P.n), dtype=np.uint64)
    st = lib().orc_decrypt(*P._args(), _p(sk_ntt, _u64p), _p(ct, _u64p), form, _p(x, _i64p), _p(xl, _u64p))
    return (x, int(st), xl) if want_limbs else (x, int(st))


def counters_reset():
    lib().orc_counters_reset()


def counters():
    t = ctypes.c_uint64(); p = ctypes.c_uint64()
    lib().orc_counters_get(ctypes.byref(t), ctypes.byref(p))
    return int(t.value), int(p.value)


# ---------------------------------------------------------------- BFV / BGV (section 4.2)
CKKS, BFV, BGV = 0, 1, 2


def keygen_scheme(P: Params, seed: int, scheme: int, t: int = 0):
    """Gen with BGV's t-scaled key error (reading A17); CKKS / BFV equal `keygen`."""
    sk = np.zeros(P.n, dtype=np.int64)
    sk_ntt = np.zeros((P.L, P.n), dtype=np.uint64)
    pk = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_keygen_scaled(*P._args(), seed, t if scheme == BGV else 1, _p(sk, _i64p), _p(sk_ntt, _u64p),
                            _p(pk, _u64p))
    return sk, sk_ntt, pk


def bfv_delta_mod(P: Params, t: int):
    return [int(lib().orc_bfv_delta_mod(P.L, _p(P.q, _u64p), t, i)) for i in range(P.L)]


def plaintext_residues(P: Params, scheme: int, t: int, m) -> np.ndarray:
    m = _i64(m)
    out = np.zeros((P.L, P.n), dtype=np.uint64)
    lib().orc_plaintext_residues(scheme, t, P.log_n, P.L, _p(P.q, _u64p), _p(m, _i64p), _p(out, _u64p))
    return out


def encrypt_general_explicit(P: Params, pk, pt_res, u, e1, e2, es: int, form: int) -> np.ndarray:
    pk, pt_res, u, e1, e2 = _u64(pk), _u64(pt_res), _i64(u), _i64(e1), _i64(e2)
    ct = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_encrypt_general_explicit(*P._args(), _p(pk, _u64p), _p(pt_res, _u64p), _p(u, _i64p), _p(e1, _i64p),
                                       _p(e2, _i64p), es, form, _p(ct, _u64p))
    return ct


def encrypt_scheme(P: Params, scheme: int, t: int, pk, m, seed: int, msg: int, form: int) -> np.ndarray:
    pk, m = _u64(pk), _i64(m)
    ct = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_encrypt_scheme(scheme, t, *P._args(), _p(pk, _u64p), _p(m, _i64p), seed, msg, form, _p(ct, _u64p))
    return ct


def precompute_cache_scheme(P: Params, scheme: int, t: int, pk, cache_seed: int, form: int) -> np.ndarray:
    pk = _u64(pk)
    cache = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_precompute_cache_scheme(scheme, t, *P._args(), _p(pk, _u64p), cache_seed, form, _p(cache, _u64p))
    return cache


def zinc_encrypt_scheme(P: Params, scheme: int, t: int, cache, form: int, m, seed: int, msg: int) -> np.ndarray:
    cache, m = _u64(cache), _i64(m)
    ct = np.zeros((2, P.L, P.n), dtype=np.uint64)
    lib().orc_zinc_encrypt_scheme(scheme, t, *P._args(), _p(cache, _u64p), form, _p(m, _i64p), seed, msg,
                                  _p(ct, _u64p))
    return ct


def crt_centered(P: Params, x_limbs) -> list:
    """x in (-Q/2, Q/2] from its residues [L][N] (plain big-integer CRT, Python ints)."""
    q = [int(v) for v in P.q]
    Q = 1
    for v in q:
        Q *= v
    coef = []
    for i, qi in enumerate(q):
        Qi = Q // qi
        coef.append(Qi * pow(Qi % qi, -1, qi))
    out = []
    xl = [[int(v) for v in row] for row in np.asarray(x_limbs)]
    for j in range(P.n):
        x = sum(xl[i][j] * coef[i] for i in range(P.L)) % Q
        out.append(x - Q if x > Q // 2 else x)
    return out, Q


def decrypt_scheme(P: Params, scheme: int, t: int, sk_ntt, ct, form: int) -> np.ndarray:
    """BFV: m = round(t.x/Q) mod t; BGV: m = x mod t; x = [c1 + c2.sk]_Q centred
    (Eq. 10 with the decoders of the original schemes)."""
    _, _, xl = decrypt(P, sk_ntt, ct, form, want_limbs=True)
    xs, Q = crt_centered(P, xl)
    if scheme == BFV:
        m = [((2 * t * x + Q) // (2 * Q)) % t for x in xs]  # round half up of t x / Q
    else:
        m = [x % t for x in xs]
    return np.array(m, dtype=np.int64)


# ---------------------------------------------------------------- Eq. 2: batched (+) and aggregation
def ct_add(P: Params, a, b) -> np.ndarray:
    a, b = _u64(a), _u64(b)
    out = np.zeros_like(a)
    count = a.size // (2 * P.L * P.n)
    lib().orc_ct_add(P.log_n, P.L, _p(P.q, _u64p), _p(a, _u64p), _p(b, _u64p), count, _p(out, _u64p))
    return out


def ct_sum(P: Params, ct) -> np.ndarray:
    ct = _u64(ct)
    out = np.zeros((2, P.L, P.n), dtype=np.uint64)
    count = ct.size // (2 * P.L * P.n)
    lib().orc_ct_sum(P.log_n, P.L, _p(P.q, _u64p), _p(ct, _u64p), count, _p(out, _u64p))
    return out


# ---------------------------------------------------------------- wide plaintexts (f3: Delta = 2^55)
def encode_i128(z, log_n: int, log_scale: int) -> np.ndarray:
    """C-6 encode with 128-bit coefficients: int64[N][2] (lo, hi) pairs."""
    re, im = _slots(z)
    m = np.zeros((1 << log_n, 2), dtype=np.int64)
    lib().orc_encode_fft_i128(_p(re, _f64p), _p(im, _f64p), log_n, log_scale, _p(m, _i64p))
    return m


def decode_i128(x, log_n: int, log_scale: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.int64)
    re = np.zeros(1 << (log_n - 1)); im = np.zeros_like(re)
    lib().orc_decode_fft_i128(_p(x, _i64p), log_n, log_scale, _p(re, _f64p), _p(im, _f64p))
    return re + 1j * im


def i128_to_int(m) -> list:
    """int64[N][2] (lo, hi) pairs -> Python ints."""
    m = np.asarray(m, dtype=np.int64)
    return [int(hi) * (1 << 64) + (int(lo) & ((1 << 64) - 1)) for lo, hi in m]


def int_to_i128(v) -> np.ndarray:
    out = np.zeros((len(v), 2), dtype=np.int64)
    for j, x in enumerate(v):
        lo = x & ((1 << 64) - 1)
        out[j, 0] = lo - (1 << 64) if lo >= (1 << 63) else lo
        out[j, 1] = x >> 64
    return out


def residues_of_ints(P: Params, v) -> np.ndarray:
    """[L][N] canonical residues of Python-int plaintext coefficients."""
    return np.array([[x % int(q) for x in v] for q in P.q], dtype=np.uint64)


def decrypt_wide(P: Params, sk_ntt, ct, form: int):
    """Eq. 10 with a two-limb CRT: x in (-q0 q1 / 2, q0 q1 / 2] from limbs 0 and 1 (Python
    ints), status 0 iff x mod q_i matches every other limb.  Returns (x ints, status)."""
    _, _, xl = decrypt(P, sk_ntt, ct, form, want_limbs=True)
    q0, q1 = int(P.q[0]), int(P.q[1])
    Q2 = q0 * q1
    inv = pow(q0, -1, q1)
    xs, st = [], 0
    for j in range(P.n):
        x0, x1 = int(xl[0][j]), int(xl[1][j])
        x = x0 + q0 * (((x1 - x0) * inv) % q1)
        if x > Q2 // 2:
            x -= Q2
        for i in range(2, P.L):
            if x % int(P.q[i]) != int(xl[i][j]):
                st = 1
        xs.append(x)
    return xs, st
