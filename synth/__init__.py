"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: only parameter-set
configuration (bit sizes and counts, i.e. workload shape) and seeded
numpy generators for slot vectors, images and conv weights.

Parameter sets (R-PRIMES):
  * ``toy``  -- BASELINE config 1: N = 2^12, 3 RNS limbs + 1 special prime.
  * ``hyp``  -- Set_hyp: N = 2^16, L+1 = 24, dnum = 6 (alpha = K = 4),
               8-byte words (Ctxt 10 MB = 2 x 10 limbs x 512 KiB at the post-boot level).
"""
from __future__ import annotations

import numpy as np

PARAMS = {
    # P:1028 (h = 192), DESIGN R-PRIMES (bit sizes, all <= 48 bits), R-SCALE (log_scale)
    "toy": dict(log_n=12, q_bits=[48, 40, 40], p_bits=[48], dnum=3, h=64, log_scale=40),
    # levels 10..23 are bootstrapping's (DESIGN R-PRIMES, R-SFFT): q_10..q_20 46 bits for EvalMod (its scale follows
    # the primes; 2^46 with digits 2^8 below P keeps the key-switch noise 2^-31 of it), q_21..q_23 48 bits for
    # CoeffToSlot's diagonals; every conv layer and block runs at levels <= 9 on the 42-bit primes (R-LEVELS)
    "hyp": dict(log_n=16, q_bits=[48] + [42] * 9 + [46] * 11 + [48] * 3, p_bits=[48] * 4, dnum=6, h=192,
                log_scale=42),
    # small full-featured set used by fast CPU tests (alpha = 2, partial last digit)
    "mini": dict(log_n=10, q_bits=[48, 40, 40, 40, 40], p_bits=[48, 48], dnum=3, h=32, log_scale=40),
    # the bootstrapping tests' chain: room for ModRaise, CoeffToSlot, EvalMod (Chebyshev depth 6
    # + 3 double angles), SlotToCoeff; small h keeps the ModRaise overflow I small (insecure, test only)
    "boot": dict(log_n=10, q_bits=[48] + [40] * 16, p_bits=[48] * 3, dnum=6, h=16, log_scale=40),
}

SEED_SK = 3        # secret-key seed of BASELINE config 1
SEED_EVK = 0x5EED_E7C
SEED_ENC = 0x5EED_E4C


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def slots_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """n real slot values ~ U(lo, hi)."""
    return rng(seed).uniform(lo, hi, size=n)


def image(seed: int, c: int, w: int) -> np.ndarray:
    """X ~ U(-1, 1)^{c x w x w}."""
    return rng(seed).uniform(-1.0, 1.0, size=(c, w, w))


def conv_weight(seed: int, co: int, ci: int, f: int) -> np.ndarray:
    """Kaiming-normal N(0, 2/(ci f^2)) conv weights."""
    return rng(seed).normal(0.0, np.sqrt(2.0 / (ci * f * f)), size=(co, ci, f, f))


def conv_bias(seed: int, co: int, scale: float = 0.1) -> np.ndarray:
    return rng(seed).uniform(-scale, scale, size=co)


def int_coeffs(seed: int, n: int, bound: int) -> np.ndarray:
    """random integer polynomial coefficients in [-bound, bound]."""
    return rng(seed).integers(-bound, bound + 1, size=n, dtype=np.int64)


def residues(seed: int, shape, moduli) -> np.ndarray:
    """uniform residues: last-but-one axis indexes the modulus list (shape[-2] == len(moduli))."""
    g = rng(seed)
    out = np.empty(shape, dtype=np.uint64)
    m = np.asarray(moduli, dtype=np.uint64)
    assert shape[-2] == len(m)
    flat = out.reshape(-1, shape[-2], shape[-1])
    for i in range(flat.shape[0]):
        for t in range(len(m)):
            flat[i, t] = g.integers(0, int(m[t]), size=shape[-1], dtype=np.uint64)
    return out
