"""Seeded synthetic input generators shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the GoCkpt method (no AdamW, no partition,
no replay). It only turns (seed, stream, step, index) counters into bit
patterns with integer hashing and exact power-of-two scalings, so the numpy
side (here) and the CUDA side (``gck_h_generate`` in the harness part of the
library) produce bit-identical inputs from the same definition:

  mix(z)   = splitmix64 finaliser:  z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
             z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31   (mod 2^64)
  h        = mix(mix(mix(seed ^ (stream * 0x9E3779B97F4A7C15)) ^ step) ^ idx)
  u24      = h >> 40                                  (24 random bits)

Distributions (DESIGN.md §"Input recipe"), all exact in their formats:
  master   "flat":   (u24 - 2^23) * 2^-23            in [-1, 1)
           "model":  (u24 - 2^23) * 2^-29            in [-2^-6, 2^-6) (matrix init scale)
  exp_avg  (warm):   (u24 - 2^23) * 2^-33            in [-2^-10, 2^-10)
  exp_avg_sq (warm): (u24 + 1) * 2^-44               in (0, 2^-20]   (strictly positive)
  grad "uniform":    bf16 of (k - 64) * 2^-6, k = h>>57  in [-1, 1)
  grad "llm":        bf16 with sign = bit 63, exponent 2^-(6+e), e = (h>>56)&15,
                     mantissa (h>>40)&0x7F  (log-uniform magnitudes 2^-21..2^-5);
                     exactly 0 when ((h>>32)&0xFF) < zero_per_256 (embedding rows
                     absent from the batch).
Streams: 1 = master, 2 = exp_avg, 3 = exp_avg_sq, 4 = gradient (step = training step).
"""

from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1

STREAM_MASTER, STREAM_M, STREAM_V, STREAM_GRAD = 1, 2, 3, 4
GRAD_UNIFORM, GRAD_LLM = 0, 1
MASTER_FLAT, MASTER_MODEL = 0, 1


def _mix_int(z: int) -> int:
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


def _mix_arr(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    z = z ^ (z >> np.uint64(31))
    return z


def hash_at(seed: int, stream: int, step: int, idx: np.ndarray) -> np.ndarray:
    """h for every global element index in idx (uint64 array)."""
    key = _mix_int(_mix_int((seed ^ ((stream * _GOLD) & MASK64)) & MASK64) ^ (step & MASK64))
    with np.errstate(over="ignore"):
        return _mix_arr(np.uint64(key) ^ np.asarray(idx, dtype=np.uint64))


def _idx(n_or_idx, offset=0):
    if np.isscalar(n_or_idx):
        return np.arange(offset, offset + int(n_or_idx), dtype=np.uint64)
    return np.asarray(n_or_idx, dtype=np.uint64)


def _u24_centered(h: np.ndarray) -> np.ndarray:
    return (h >> np.uint64(40)).astype(np.int64) - (1 << 23)


def master(seed: int, n_or_idx, offset: int = 0, mode: int = MASTER_FLAT) -> np.ndarray:
    h = hash_at(seed, STREAM_MASTER, 0, _idx(n_or_idx, offset))
    scale = 2.0 ** -23 if mode == MASTER_FLAT else 2.0 ** -29
    return (_u24_centered(h).astype(np.float64) * scale).astype(np.float32)  # exact


def exp_avg(seed: int, n_or_idx, offset: int = 0) -> np.ndarray:
    h = hash_at(seed, STREAM_M, 0, _idx(n_or_idx, offset))
    return (_u24_centered(h).astype(np.float64) * 2.0 ** -33).astype(np.float32)  # exact


def exp_avg_sq(seed: int, n_or_idx, offset: int = 0) -> np.ndarray:
    h = hash_at(seed, STREAM_V, 0, _idx(n_or_idx, offset))
    return (((h >> np.uint64(40)).astype(np.float64) + 1.0) * 2.0 ** -44).astype(np.float32)  # exact


def grad_bits(seed: int, step: int, n_or_idx, offset: int = 0, mode: int = GRAD_LLM,
              zero_per_256: int = 4) -> np.ndarray:
    """bf16 gradient bit patterns (uint16) of training step `step`."""
    h = hash_at(seed, STREAM_GRAD, step, _idx(n_or_idx, offset))
    if mode == GRAD_UNIFORM:
        k = (h >> np.uint64(57)).astype(np.int64) - 64
        f = (k.astype(np.float64) * 2.0 ** -6).astype(np.float32)      # exact, <= 7 significant bits
        return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)  # exact truncation
    sign = ((h >> np.uint64(63)) & np.uint64(1)).astype(np.uint32)
    e = ((h >> np.uint64(56)) & np.uint64(15)).astype(np.uint32)
    mant = ((h >> np.uint64(40)) & np.uint64(0x7F)).astype(np.uint32)
    bits = (sign << np.uint32(15)) | ((np.uint32(127 - 6) - e) << np.uint32(7)) | mant
    zero = ((h >> np.uint64(32)) & np.uint64(0xFF)) < np.uint64(zero_per_256)
    bits[zero] = 0
    return bits.astype(np.uint16)


def warm_state(seed: int, n_or_idx, offset: int = 0, mode: int = MASTER_FLAT):
    """A synthetic mid-training state S(t0): (master, exp_avg, exp_avg_sq)."""
    return (master(seed, n_or_idx, offset, mode), exp_avg(seed, n_or_idx, offset),
            exp_avg_sq(seed, n_or_idx, offset))


def cold_state(seed: int, n_or_idx, offset: int = 0, mode: int = MASTER_FLAT):
    """S(0): generated master, zero moments."""
    p = master(seed, n_or_idx, offset, mode)
    return p, np.zeros_like(p), np.zeros_like(p)
