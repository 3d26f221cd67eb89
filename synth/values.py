"""Seeded synthetic gradient values (test/bench infrastructure, no method arithmetic).

Recipe (stated in DESIGN.md "Input recipe"): the values of tensor t on rank r at
step s come from numpy's PCG64 seeded with SeedSequence([seed, s, r, t]).
Each tensor has a fixed scale sigma_t = 10**U(-4, -1) drawn from
SeedSequence([seed, t, 0x5167]) so magnitudes differ across tensors like real
per-layer gradients.  Distributions:

  D1  Gaussian N(0, sigma_t^2)
  D2  Laplace(0, sigma_t)                     (heavy tail)
  D3  D1 rounded to bfloat16                  (heavy magnitude ties)
  D4  adversarial: all-equal |x| with random signs, all zeros, a single spike,
      a +0/-0 mix, denormals (chosen per tensor by `mode`)

The arrays are generated on the host; the CUDA path receives them by upload and
the oracle receives the same arrays, so both sides see identical bits.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 220514465
D4_MODES = ("equal", "zeros", "spike", "pm0", "denormal", "mixed")


def sigma(seed: int, tensor: int) -> np.float32:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, tensor, 0x5167])))
    return np.float32(10.0 ** rng.uniform(-4.0, -1.0))


def _rng(seed, step, rank, tensor):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, step, rank, tensor])))


def _bf16_round(x: np.ndarray) -> np.ndarray:
    u = x.view(np.uint32).astype(np.uint64)
    # round-to-nearest-even on the upper 16 bits (finite inputs)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def gradient(n: int, seed: int = BASE_SEED, step: int = 0, rank: int = 0, tensor: int = 0,
             dist: str = "D1", mode: str = "mixed") -> np.ndarray:
    """fp32 array of length n (contiguous, C order)."""
    rng = _rng(seed, step, rank, tensor)
    s = sigma(seed, tensor)
    if dist == "D1":
        x = rng.standard_normal(n, dtype=np.float32) * s
    elif dist == "D2":
        x = rng.laplace(0.0, float(s), n).astype(np.float32)
    elif dist == "D3":
        x = _bf16_round(rng.standard_normal(n, dtype=np.float32) * s)
    elif dist == "D4":
        x = _adversarial(n, rng, s, mode)
    else:
        raise ValueError(dist)
    return np.ascontiguousarray(x, dtype=np.float32)


def _adversarial(n, rng, s, mode):
    if mode == "mixed":
        # cycle through the single modes in blocks of 97 elements
        out = np.empty(n, np.float32)
        singles = D4_MODES[:-1]
        for b, lo in enumerate(range(0, n, 97)):
            hi = min(n, lo + 97)
            out[lo:hi] = _adversarial(hi - lo, rng, s, singles[b % len(singles)])
        return out
    if mode == "equal":
        sign = rng.integers(0, 2, n).astype(np.float32) * 2 - 1
        return (sign * s).astype(np.float32)
    if mode == "zeros":
        return np.zeros(n, np.float32)
    if mode == "spike":
        x = np.zeros(n, np.float32)
        if n:
            x[rng.integers(0, n)] = np.float32(1000.0) * s
        return x
    if mode == "pm0":
        x = np.where(rng.integers(0, 2, n) == 0, np.float32(0.0), np.float32(-0.0)).astype(np.float32)
        nz = rng.integers(0, 2, n) == 1
        x[nz & (rng.integers(0, 8, n) == 0)] = s
        return x
    if mode == "denormal":
        bits = rng.integers(1, 1 << 23, n).astype(np.uint32) | (rng.integers(0, 2, n).astype(np.uint32) << 31)
        return bits.view(np.float32).copy()
    raise ValueError(mode)


def rank_gradients(numels, seed=BASE_SEED, step=0, rank=0, dist="D1", mode="mixed"):
    """One gradient per tensor of a model on one rank."""
    return [gradient(n, seed, step, rank, t, dist, mode) for t, n in enumerate(numels)]
