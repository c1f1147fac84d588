"""Deterministic synthetic workloads (SURVEY.md 8(d) "Synthetic inputs").

Counter-based, integer-only generator so the device (csrc/store.cu
``synth_fill_kernel``) and the host (this module, numpy) produce bit-identical
values without sharing state:

* context value (record i, dim k) = (u0 + u1 + u2 + u3 - 8190) * 2**-11 where the
  u's are four 12-bit fields of splitmix64(seed, i * d + k): an Irwin-Hall(4)
  approximation of N(0, 1.155^2), |x| <= 4, a multiple of 2**-11 -- exact in
  fp32, and every running sum / sum of squares of up to 2**27 records is exact
  in fp64, so reduction order cannot change the store statistics;
* reward = (2**13 + low 20 bits) * 2**-20, i.e. U[2**-7, 1 + 2**-7), always > 0
  (nothing is gated out) and fp32-exact;
* round = global index.

The "clustered" variant adds one of 64 centres (same generator, stream 0xC1u)
scaled by 2 so retrieval has real structure.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return np.uint64((seed * 0x100000001B3 + stream * 0x9E3779B1) & 0xFFFFFFFFFFFFFFFF)


def contexts(seed: int, start: int, count: int, d: int, clustered: bool = False) -> np.ndarray:
    """[count, d] float64 (fp32-exact) contexts of records start..start+count-1."""
    idx = (np.arange(start, start + count, dtype=np.uint64)[:, None] * np.uint64(d)
           + np.arange(d, dtype=np.uint64)[None, :])
    with np.errstate(over="ignore"):
        h = splitmix64(idx ^ _key(seed, 1))
    m = np.uint64(0xFFF)
    s = ((h & m) + ((h >> np.uint64(12)) & m) + ((h >> np.uint64(24)) & m)
         + ((h >> np.uint64(36)) & m)).astype(np.int64)
    x = (s - 8190).astype(np.float64) * 2.0 ** -11
    if clustered:
        cid = (splitmix64(np.arange(start, start + count, dtype=np.uint64) ^ _key(seed, 0xC1))
               % np.uint64(64)).astype(np.int64)
        centres = contexts(seed ^ 0x5EED, 0, 64, d) * 2.0
        x = x + centres[cid]
    return x


def rewards(seed: int, start: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = splitmix64(np.arange(start, start + count, dtype=np.uint64) ^ _key(seed, 2))
    k = (h & np.uint64(0xFFFFF)).astype(np.int64)
    return (k + 8192).astype(np.float64) * 2.0 ** -20


def rounds(start: int, count: int) -> np.ndarray:
    return np.arange(start, start + count, dtype=np.int64).astype(np.int32)


def queries(seed: int, count: int, d: int, clustered: bool = False) -> np.ndarray:
    return contexts(seed ^ 0x0DDBA11, 0, count, d, clustered)


def tuples(seed: int, T: int, K: int, dist: str = "uniform") -> np.ndarray:
    """[T, K] objective tuples in [0, 1], multiples of 2**-24 (8(d) config 3).

    uniform | anti (sum ~= 1 +- 0.01) | corr | grid (1/256 grid: ties/duplicates)
    """
    idx = (np.arange(T, dtype=np.uint64)[:, None] * np.uint64(K)
           + np.arange(K, dtype=np.uint64)[None, :])
    with np.errstate(over="ignore"):
        h = splitmix64(idx ^ _key(seed, 3))
    u = (h >> np.uint64(40)).astype(np.float64) * 2.0 ** -24  # [0,1) on the 2^-24 grid
    if dist == "uniform":
        return u
    if dist == "grid":
        return np.floor(u * 256.0) / 256.0
    if dist == "anti":
        # project onto the simplex sum = 1 with +-0.01 jitter, then re-grid
        w = u / np.maximum(u.sum(axis=1, keepdims=True), 1e-12)
        j = (h & np.uint64(0xFFFF)).astype(np.float64)[:, :1] * 2.0 ** -16
        x = w * (0.99 + 0.02 * j)
        return np.clip(np.floor(x * 2.0 ** 24) / 2.0 ** 24, 0.0, 1.0)
    if dist == "corr":
        base = u[:, :1]
        x = 0.8 * base + 0.2 * u
        return np.floor(x * 2.0 ** 24) / 2.0 ** 24
    raise ValueError(dist)
