"""paper_2408_07304_b200 -- B200 (sm_100a) hot path of arXiv 2408.07304 ("Zinc").

Thin Python binding of ``libzinc.so`` (C ABI in ``include/zinc.h``): argument
marshalling only.  Every step of the encryption path runs in the library's CUDA
kernels; PyTorch supplies device memory and streams.  There is no CPU fallback:
if the shared library is missing or cannot be loaded, importing this package's
functions raises.

Function names follow the ABI (``zinc_keygen``, ``zinc_precompute_cache``,
``zinc_encrypt_batch``, ``ckks_encrypt_batch``, ``ckks_decrypt_batch``, ...).
Tensors: uint64 ciphertexts ``[B, 2, L, N]``, keys ``[2, L, N]``, secret key
``[L, N]``; int64 plaintexts ``[B, N]``; float64 slots ``[B, N/2]`` (real) or
``[B, N/2, 2]`` (complex).
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "NTT", "COEFF", "PT_COEFF_I64", "PT_SLOTS_F64", "PT_SLOTS_C128", "ZincError", "Context", "lib",
    "zinc_keygen", "zinc_precompute_cache", "zinc_encrypt_batch", "ckks_encrypt_batch",
    "ckks_decrypt_batch", "ckks_encode_batch", "zinc_ntt_forward", "zinc_ntt_inverse",
    "zinc_debug_sample", "zinc_int_peak", "zinc_ct_add_batch", "zinc_ct_sum_batch", "zinc_encrypt_batch_host", "launch_count",
    "launch_count_reset", "tune", "TUNE_COEFF_MSGS_PER_CTA", "TUNE_ENCODE_CHUNK_BYTES", "TUNE_PDL", "TUNE_L2_PREFETCH",
    "TUNE_NTT_CHUNK_MSGS", "TUNE_SPLIT", "TUNE_SMALL_ENCODE", "TUNE_PT_IN_CT", "TUNE_SMALL_CLUSTER", "TUNE_M_DEINT", "BFLY_CT", "BFLY_CT_NR", "BFLY_CT_A", "BFLY_GS", "LIB_PATH", "EXPORTED_SYMBOLS", "profile_enable", "profile_read", "KERNEL_NAMES",
]

NTT, COEFF = 0, 1
CKKS, BFV, BGV = 0, 1, 2
PT_COEFF_I64, PT_SLOTS_F64, PT_SLOTS_C128, PT_COEFF_I128 = 0, 1, 2, 3
PATH_ZINC, PATH_VANILLA = 0, 1

LIB_PATH = os.environ.get("ZINC_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libzinc.so")

# every symbol include/zinc.h declares
EXPORTED_SYMBOLS = (
    "zinc_ctx_create", "zinc_ctx_destroy", "zinc_ctx_moduli", "zinc_ctx_info", "zinc_keygen",
    "zinc_precompute_cache", "zinc_encrypt_batch", "ckks_encrypt_batch", "ckks_decrypt_batch",
    "ckks_encode_batch", "zinc_ntt_forward", "zinc_ntt_inverse", "zinc_debug_sample", "zinc_int_peak",
    "zinc_encrypt_batch_host", "zinc_launch_count", "zinc_launch_count_reset", "zinc_last_error",
    "zinc_profile_enable", "zinc_profile_read", "zinc_kernel_name", "zinc_tune", "zinc_ctx_create_scheme",
    "zinc_ctx_scheme", "zinc_ct_add_batch", "zinc_ct_sum_batch", "ckks_encode_batch_wide", "ckks_decrypt_batch_wide",
)
KERNEL_NAMES = ("zinc_coeff_kernel", "zinc_ntt_kernel", "vanilla_kernel", "keygen_kernel", "encode_kernel",
                "decrypt_kernel", "decode_kernel", "ntt_kernel", "sample_kernel", "int_peak_kernel",
                "bfv_scale_kernel", "ct_add_kernel", "ct_sum_kernel", "lift_kernel", "pt_add_kernel",
                "shoup_prep_kernel")
# zinc_int_peak butterfly variants (include/zinc.h)
BFLY_CT, BFLY_CT_NR, BFLY_CT_A, BFLY_GS = 0, 1, 2, 3


class ZincError(RuntimeError):
    pass


_c = ctypes
_vp, _u64, _i32, _sz = _c.c_void_p, _c.c_uint64, _c.c_int, _c.c_size_t
_SIGS = {
    "zinc_ctx_create": [_i32, _i32, _c.POINTER(_c.c_int), _i32, _i32, _c.POINTER(_vp)],
    "zinc_ctx_destroy": [_vp],
    "zinc_ctx_moduli": [_vp, _c.POINTER(_u64), _c.POINTER(_u64)],
    "zinc_ctx_info": [_vp, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)],
    "zinc_keygen": [_vp, _u64, _vp, _vp, _vp, _vp],
    "zinc_precompute_cache": [_vp, _vp, _u64, _i32, _vp, _vp],
    "zinc_encrypt_batch": [_vp, _vp, _i32, _i32, _vp, _sz, _u64, _u64, _vp, _vp],
    "ckks_encrypt_batch": [_vp, _vp, _i32, _i32, _vp, _sz, _u64, _u64, _vp, _vp],
    "ckks_decrypt_batch": [_vp, _vp, _i32, _vp, _sz, _vp, _vp, _vp, _vp],
    "ckks_encode_batch": [_vp, _i32, _vp, _sz, _vp, _vp],
    "zinc_ntt_forward": [_vp, _vp, _sz, _vp],
    "zinc_ntt_inverse": [_vp, _vp, _sz, _vp],
    "zinc_debug_sample": [_vp, _i32, _u64, _u64, _i32, _sz, _vp, _vp],
    "zinc_int_peak": [_vp, _i32, _i32, _i32, _vp, _c.POINTER(_c.c_double), _vp],
    "zinc_encrypt_batch_host": [_vp, _i32, _vp, _i32, _i32, _vp, _sz, _u64, _u64, _vp, _sz, _vp],
    "zinc_profile_enable": [_i32],
    "zinc_profile_read": [_c.POINTER(_c.c_double), _c.POINTER(_u64)],
    "zinc_tune": [_i32, _c.c_longlong, _c.POINTER(_c.c_longlong)],
    "zinc_ctx_create_scheme": [_i32, _i32, _c.POINTER(_c.c_int), _i32, _u64, _i32, _i32, _c.POINTER(_vp)],
    "zinc_ctx_scheme": [_vp, _c.POINTER(_c.c_int), _c.POINTER(_u64)],
    "zinc_ct_add_batch": [_vp, _vp, _vp, _sz, _vp, _vp],
    "zinc_ct_sum_batch": [_vp, _vp, _sz, _vp, _vp],
    "ckks_encode_batch_wide": [_vp, _i32, _vp, _sz, _vp, _vp],
    "ckks_decrypt_batch_wide": [_vp, _vp, _i32, _vp, _sz, _vp, _vp, _vp, _vp],
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libzinc.so (raises ZincError if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ZincError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _c.c_int
        L.zinc_last_error.restype = _c.c_char_p
        L.zinc_last_error.argtypes = []
        L.zinc_kernel_name.restype = _c.c_char_p
        L.zinc_kernel_name.argtypes = [_i32]
        L.zinc_launch_count.restype = _u64
        L.zinc_launch_count.argtypes = []
        L.zinc_launch_count_reset.restype = None
        L.zinc_launch_count_reset.argtypes = []
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().zinc_last_error().decode(errors="replace")
        raise ZincError(f"{what}: status {rc}: {msg}")


def _ptr(t):
    """Device address of a contiguous tensor (or an int address) as a plain int: the
    argtypes (c_void_p) convert it, so no ctypes object is built per argument."""
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ZincError("tensor must be contiguous")
        return t.data_ptr()
    return int(t)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream=None):
    """cudaStream_t of `stream`, else of torch's current stream on the current device (read
    through torch's raw-stream accessor: about a microsecond less per call than building a
    torch.cuda.Stream object on the small-batch latency path)."""
    if stream is None:
        if _raw_stream is not None:
            return _raw_stream(torch.cuda.current_device())
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Context:
    """A zinc_ctx: ring degree 2^log_n, RNS primes of the given bit sizes (C-1),
    scale 2^log_scale, bound to CUDA device `device`; `scheme` CKKS (default),
    BFV or BGV with plaintext modulus `t`."""

    def __init__(self, log_n: int, bits, log_scale: int, device: int = 0, scheme: int = 0, t: int = 0):
        arr = (ctypes.c_int * len(bits))(*[int(b) for b in bits])
        h = ctypes.c_void_p()
        torch.cuda.init()
        _check(lib().zinc_ctx_create_scheme(log_n, len(bits), arr, scheme, t, log_scale, device, ctypes.byref(h)),
               "zinc_ctx_create_scheme")
        self.scheme, self.t = scheme, t
        self._h = h
        self.log_n, self.L, self.log_scale, self.device = log_n, len(bits), log_scale, device
        self.n = 1 << log_n
        q = (ctypes.c_uint64 * self.L)()
        psi = (ctypes.c_uint64 * self.L)()
        _check(lib().zinc_ctx_moduli(h, q, psi), "zinc_ctx_moduli")
        self.q = [int(x) for x in q]
        self.psi = [int(x) for x in psi]

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.zinc_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # allocation helpers (torch owns device memory)
    def dev(self):
        return torch.device("cuda", self.device)

    def empty_ct(self, batch: int) -> torch.Tensor:
        return torch.empty((batch, 2, self.L, self.n), dtype=torch.uint64, device=self.dev())

    def empty_key(self) -> torch.Tensor:
        return torch.empty((2, self.L, self.n), dtype=torch.uint64, device=self.dev())


def _as_pt(pt: torch.Tensor) -> torch.Tensor:
    """complex128 slots [B, N/2] travel as their float64 (re, im) view [B, N/2, 2]."""
    return torch.view_as_real(pt) if pt.is_complex() else pt


def _kind_of(pt: torch.Tensor) -> int:
    if pt.dtype == torch.int64:
        return PT_COEFF_I128 if pt.dim() == 3 else PT_COEFF_I64
    if pt.dtype == torch.float64:
        return PT_SLOTS_C128 if pt.dim() == 3 else PT_SLOTS_F64
    raise ZincError(f"unsupported plaintext dtype {pt.dtype}")


def zinc_keygen(ctx: Context, seed: int, stream=None):
    """Gen (Eq. 7). Returns (sk_ntt [L,N] u64, sk_coeff [N] i8, pk_ntt [2,L,N] u64)."""
    sk = torch.empty((ctx.L, ctx.n), dtype=torch.uint64, device=ctx.dev())
    skc = torch.empty((ctx.n,), dtype=torch.int8, device=ctx.dev())
    pk = ctx.empty_key()
    _check(lib().zinc_keygen(ctx.handle, seed, _ptr(sk), _ptr(skc), _ptr(pk), _stream(stream)), "zinc_keygen")
    return sk, skc, pk


def zinc_precompute_cache(ctx: Context, pk_ntt: torch.Tensor, seed: int, form: int, out=None, stream=None):
    """Zinc precomputation: Enc(0) in `form`. Returns [2,L,N] u64."""
    cache = ctx.empty_key() if out is None else out
    _check(lib().zinc_precompute_cache(ctx.handle, _ptr(pk_ntt), seed, form, _ptr(cache), _stream(stream)),
           "zinc_precompute_cache")
    return cache


def zinc_encrypt_batch(ctx: Context, cache: torch.Tensor, form: int, pt: torch.Tensor, seed: int,
                       msg_base: int = 0, out=None, stream=None):
    """Enc_z (Algorithm 1) of a batch of plaintexts (int64 [B,N] or slots). Returns [B,2,L,N] u64."""
    pt = _as_pt(pt)
    b = pt.shape[0]
    ct = ctx.empty_ct(b) if out is None else out
    _check(lib().zinc_encrypt_batch(ctx.handle, _ptr(cache), form, _kind_of(pt), _ptr(pt), b, seed, msg_base,
                                    _ptr(ct), _stream(stream)), "zinc_encrypt_batch")
    return ct


def ckks_encrypt_batch(ctx: Context, pk_ntt: torch.Tensor, form: int, pt: torch.Tensor, seed: int,
                       msg_base: int = 0, out=None, stream=None):
    """Vanilla Enc (Eq. 8, reading A1) of a batch. Returns [B,2,L,N] u64."""
    pt = _as_pt(pt)
    b = pt.shape[0]
    ct = ctx.empty_ct(b) if out is None else out
    _check(lib().ckks_encrypt_batch(ctx.handle, _ptr(pk_ntt), form, _kind_of(pt), _ptr(pt), b, seed, msg_base,
                                    _ptr(ct), _stream(stream)), "ckks_encrypt_batch")
    return ct


def ckks_decrypt_batch(ctx: Context, sk_ntt: torch.Tensor, form: int, ct: torch.Tensor, slots: bool = True,
                       stream=None):
    """Dec (Eq. 10). Returns (coeff int64 [B,N], status int32 [B], slots complex128 [B,N/2] or None)."""
    b = ct.shape[0]
    coeff = torch.empty((b, ctx.n), dtype=torch.int64, device=ctx.dev())
    status = torch.empty((b,), dtype=torch.int32, device=ctx.dev())
    slots = slots and ctx.scheme == CKKS  # BFV / BGV: coeff = m in [0, t), no slots
    wide = ctx.scheme == CKKS and ctx.log_scale >= 48  # 128-bit coefficients: ckks_decrypt_batch_wide
    if wide:
        coeff = None
    z = torch.empty((b, ctx.n // 2, 2), dtype=torch.float64, device=ctx.dev()) if slots else None
    _check(lib().ckks_decrypt_batch(ctx.handle, _ptr(sk_ntt), form, _ptr(ct), b, _ptr(z), _ptr(coeff), _ptr(status),
                                    _stream(stream)), "ckks_decrypt_batch")
    zc = torch.view_as_complex(z) if slots else None
    return coeff, status, zc


def ckks_encode_batch_wide(ctx: Context, slots: torch.Tensor, out=None, stream=None):
    """Encode slots (C-6) into 128-bit coefficients. Returns int64 [B,N,2] (lo, hi)."""
    slots = _as_pt(slots)
    b = slots.shape[0]
    m = torch.empty((b, ctx.n, 2), dtype=torch.int64, device=ctx.dev()) if out is None else out
    _check(lib().ckks_encode_batch_wide(ctx.handle, _kind_of(slots), _ptr(slots), b, _ptr(m), _stream(stream)),
           "ckks_encode_batch_wide")
    return m


def ckks_decrypt_batch_wide(ctx: Context, sk_ntt: torch.Tensor, form: int, ct: torch.Tensor, slots: bool = True,
                            stream=None):
    """Dec with a two-limb CRT (f3). Returns (x int64 [B,N,2] (lo, hi), status int32 [B], slots or None)."""
    b = ct.shape[0]
    coeff = torch.empty((b, ctx.n, 2), dtype=torch.int64, device=ctx.dev())
    status = torch.empty((b,), dtype=torch.int32, device=ctx.dev())
    z = torch.empty((b, ctx.n // 2, 2), dtype=torch.float64, device=ctx.dev()) if slots else None
    _check(lib().ckks_decrypt_batch_wide(ctx.handle, _ptr(sk_ntt), form, _ptr(ct), b, _ptr(z), _ptr(coeff),
                                         _ptr(status), _stream(stream)), "ckks_decrypt_batch_wide")
    return coeff, status, (torch.view_as_complex(z) if slots else None)


def ckks_encode_batch(ctx: Context, slots: torch.Tensor, out=None, stream=None):
    """Encode slots (C-6). Returns int64 [B,N]."""
    slots = _as_pt(slots)
    b = slots.shape[0]
    m = torch.empty((b, ctx.n), dtype=torch.int64, device=ctx.dev()) if out is None else out
    _check(lib().ckks_encode_batch(ctx.handle, _kind_of(slots), _ptr(slots), b, _ptr(m), _stream(stream)),
           "ckks_encode_batch")
    return m


def zinc_ct_add_batch(ctx: Context, x: torch.Tensor, y: torch.Tensor, out=None, stream=None):
    """Eq. 2: [x + y]_q for ciphertext batches [B,2,L,N]."""
    out = torch.empty_like(x) if out is None else out
    _check(lib().zinc_ct_add_batch(ctx.handle, _ptr(x), _ptr(y), x.shape[0], _ptr(out), _stream(stream)),
           "zinc_ct_add_batch")
    return out


def zinc_ct_sum_batch(ctx: Context, ct: torch.Tensor, out=None, stream=None):
    """Aggregation: the sum of a ciphertext batch [B,2,L,N] -> [2,L,N]."""
    out = ctx.empty_key() if out is None else out
    _check(lib().zinc_ct_sum_batch(ctx.handle, _ptr(ct), ct.shape[0], _ptr(out), _stream(stream)),
           "zinc_ct_sum_batch")
    return out


def zinc_ntt_forward(ctx: Context, data: torch.Tensor, stream=None):
    """In-place forward NTT (C-3) of uint64 [count, L, N]."""
    _check(lib().zinc_ntt_forward(ctx.handle, _ptr(data), data.numel() // (ctx.L * ctx.n), _stream(stream)),
           "zinc_ntt_forward")
    return data


def zinc_ntt_inverse(ctx: Context, data: torch.Tensor, stream=None):
    _check(lib().zinc_ntt_inverse(ctx.handle, _ptr(data), data.numel() // (ctx.L * ctx.n), _stream(stream)),
           "zinc_ntt_inverse")
    return data


def zinc_debug_sample(ctx: Context, tag: int, seed: int, msg: int, limb: int, n: int, stream=None):
    dt = torch.uint64 if tag == 3 else torch.int64
    out = torch.empty((n,), dtype=dt, device=ctx.dev())
    _check(lib().zinc_debug_sample(ctx.handle, tag, seed, msg, limb, n, _ptr(out), _stream(stream)),
           "zinc_debug_sample")
    return out


def zinc_int_peak(ctx: Context, blocks: int, iters: int, sink: torch.Tensor, variant: int = BFLY_CT,
                  stream=None) -> float:
    """K11: launch `blocks` x 256 threads of `iters` x 8 register-resident butterflies of
    `variant` (BFLY_*); returns the number of butterflies launched."""
    bf = ctypes.c_double()
    _check(lib().zinc_int_peak(ctx.handle, variant, blocks, iters, _ptr(sink), ctypes.byref(bf), _stream(stream)),
           "zinc_int_peak")
    return bf.value


def zinc_encrypt_batch_host(ctx: Context, path: int, key: torch.Tensor, form: int, pt_host: torch.Tensor,
                            seed: int, msg_base: int, ct_host: torch.Tensor, chunk: int = 256, stream=None):
    """Host-buffer (end-to-end) encryption: pt_host / ct_host are CPU tensors (pinned for speed).
    The call orders itself after the work queued on `stream` (default: torch's current stream)."""
    pt_host = _as_pt(pt_host)
    if pt_host.is_cuda or ct_host.is_cuda:
        raise ZincError("zinc_encrypt_batch_host takes host tensors")
    _check(lib().zinc_encrypt_batch_host(ctx.handle, path, _ptr(key), form, _kind_of(pt_host), _ptr(pt_host),
                                         pt_host.shape[0], seed, msg_base, _ptr(ct_host), chunk, _stream(stream)),
           "zinc_encrypt_batch_host")
    return ct_host


def profile_enable(on: bool = True):
    """Start (clear) / stop per-kernel CUDA-event tracing inside the library."""
    _check(lib().zinc_profile_enable(1 if on else 0), "zinc_profile_enable")


def profile_read() -> dict:
    """{kernel name: (total device ms, launches)} since profile_enable(True)."""
    n = len(KERNEL_NAMES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_uint64 * n)()
    _check(lib().zinc_profile_read(ms, cnt), "zinc_profile_read")
    return {KERNEL_NAMES[i]: (float(ms[i]), int(cnt[i])) for i in range(n) if cnt[i]}


TUNE_COEFF_MSGS_PER_CTA, TUNE_ENCODE_CHUNK_BYTES, TUNE_PDL, TUNE_L2_PREFETCH, TUNE_NTT_CHUNK_MSGS = 0, 1, 2, 3, 4
TUNE_SPLIT, TUNE_SMALL_ENCODE, TUNE_PT_IN_CT, TUNE_SMALL_CLUSTER, TUNE_M_DEINT = 5, 6, 7, 8, 9


def tune(knob: int, value: int) -> int:
    """Set a launch-geometry knob (results never change); returns the previous value."""
    old = ctypes.c_longlong()
    _check(lib().zinc_tune(knob, value, ctypes.byref(old)), "zinc_tune")
    return old.value


def launch_count() -> int:
    return int(lib().zinc_launch_count())


def launch_count_reset():
    lib().zinc_launch_count_reset()
