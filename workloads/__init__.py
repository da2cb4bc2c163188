"""Seeded synthetic workloads C1..C5 (BASELINE.json ``configs``).

This module holds NONE of the method's arithmetic: no primes, no transforms,
no sampling of the scheme's randomness.  It only states each configuration's
shape (ring degree, limb bit sizes, scale, batch, slot distribution) and
generates the slot / integer-plaintext inputs from numpy seeds, so that the
CUDA path (bench.py, the binding's users) and the oracle (tests) consume the
identical inputs.  Neither side is imported here.

Slot recipe: message ``b`` of config ``cfg`` draws from
``numpy.random.default_rng([cfg.id, b])``.  The paper's datasets
are not in the container; these synthetic inputs stand in for them.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    id: int
    log_n: int
    bits: tuple
    log_scale: int
    batch: int
    dist: str            # "uniform", "c3_mix", "complex_uniform"
    complex_slots: bool = False
    batches: tuple = field(default=())   # C5 sweep
    key_seed: int = 0
    cache_seed: int = 0
    enc_seed: int = 0

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def slots(self) -> int:
        return self.n // 2

    @property
    def L(self) -> int:
        return len(self.bits)

    def tolerance(self) -> float:
        """Decode tolerance fixed by BASELINE.json north_star: 1e-4 at 2^40, 1e-3 at 2^30."""
        return 1e-4 if self.log_scale >= 40 else 1e-3


def _cfg(name, id_, log_n, bits, log_scale, batch, dist, complex_slots=False, batches=()):
    return Config(name, id_, log_n, tuple(bits), log_scale, batch, dist, complex_slots, tuple(batches),
                  key_seed=0x5EED0000 + id_, cache_seed=0xCAC4E000 + id_, enc_seed=0xE4C00000 + id_)


PAPER_BITS = (56,) + (55,) * 15  # BFVDefault(32768), 881-bit Q; the 56-bit prime is limb 0 (C-10)

CONFIGS = {
    "C1": _cfg("C1", 1, 12, [36] * 3, 30, 256, "uniform"),
    "C2": _cfg("C2", 2, 13, [60, 40, 40, 60], 40, 4096, "uniform"),
    "C3": _cfg("C3", 3, 14, [54] * 8, 40, 16384, "c3_mix"),
    "C4": _cfg("C4", 4, 15, [55] * 16, 40, 8192, "complex_uniform", complex_slots=True),
    "C5": _cfg("C5", 5, 14, [54] * 8, 40, 4096, "uniform", batches=(1, 16, 256, 4096, 65536)),
    # the paper's own parameters (N = 2^15, Delta = 2^55) with
    # stand-ins shaped like Table 2's datasets (the data are not in the container):
    # one ciphertext per Covid-19 day (16 metrics), per Bitcoin value, per hg38 row (values < 2^9,
    # PAPER.md:396).  Counts are the paper's; value recipes are stated in message_slots.
    "P_covid": _cfg("P_covid", 11, 15, PAPER_BITS, 55, 341, "covid"),
    "P_bitcoin": _cfg("P_bitcoin", 12, 15, PAPER_BITS, 55, 1086, "bitcoin"),
    "P_hg38": _cfg("P_hg38", 13, 15, PAPER_BITS, 55, 34424, "hg38"),
}


def message_slots(cfg: Config, b: int) -> np.ndarray:
    """Slots of global message index ``b``: float64[N/2] or complex128[N/2]."""
    rng = np.random.default_rng([cfg.id, b])
    s = cfg.slots
    if cfg.dist == "uniform":
        return rng.uniform(-1.0, 1.0, s)
    if cfg.dist == "c3_mix":
        # reading A13: messages [0, B/2) uniform on [-1, 1], [B/2, B) N(0,1) clipped to +-4
        if (b % cfg.batch) < cfg.batch // 2:
            return rng.uniform(-1.0, 1.0, s)
        return np.clip(rng.standard_normal(s), -4.0, 4.0)
    if cfg.dist == "covid":      # 16 daily counts in the first slots, rest zero
        out = np.zeros(s)
        out[:16] = rng.integers(0, 1 << 20, 16)
        return out
    if cfg.dist == "bitcoin":    # one price-like value (needs 32 Rache pivots: < 2^32) in slot 0
        out = np.zeros(s)
        out[0] = rng.integers(1 << 20, 1 << 32)
        return out
    if cfg.dist == "hg38":       # one row of small genomic counts (< 2^9) in the first slots
        out = np.zeros(s)
        out[:8] = rng.integers(0, 1 << 9, 8)
        return out
    if cfg.dist == "complex_uniform":
        re = rng.uniform(-1.0, 1.0, s)
        im = rng.uniform(-1.0, 1.0, s)
        return re + 1j * im
    raise ValueError(cfg.dist)


def slots_batch(cfg: Config, start: int, count: int) -> np.ndarray:
    """Slots of messages [start, start+count): float64[count][N/2] (complex128 for C4)."""
    dt = np.complex128 if cfg.complex_slots else np.float64
    out = np.empty((count, cfg.slots), dtype=dt)
    for i in range(count):
        out[i] = message_slots(cfg, start + i)
    return out


def int_plaintexts(log_n: int, count: int, seed: int, bound_bits: int = 45) -> np.ndarray:
    """Random integer plaintext polynomials int64[count][N] with |m| < 2^bound_bits,
    for the bit-exact contract (ciphertexts from the same int64 m and seed)."""
    rng = np.random.default_rng([0x1D7, seed])
    lim = 1 << bound_bits
    return rng.integers(-lim + 1, lim, size=(count, 1 << log_n), dtype=np.int64)
