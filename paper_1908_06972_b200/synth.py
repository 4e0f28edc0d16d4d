"""Seeded synthetic input generators shared by the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws random numbers
(numpy PCG64, seeded) in the shapes and distributions of the paper's workloads.
Random numbers the method consumes (secret key, key/encryption randomness) are
drawn here and passed to BOTH the oracle and the CUDA path as inputs, so neither
side depends on the other's sampler (task rule 3; recipe in DESIGN.md "Inputs").

Distributions (P:138 SETUP, P:399 sigma = 3.2, reading A2/A3):
  * uniform residues mod q, drawn independently per limb;
  * binary polynomials (secret s, ephemeral u) from {0, 1};
  * "Gaussian" errors: round(Normal(0, sigma)) clipped to |x| <= 19 (6 sigma);
  * real slot vectors U[-1, 1];
  * PrivFT bags: w ~ U{50..600} tokens with Zipf(1.1) ids over [0, m).
"""
from __future__ import annotations

import numpy as np

SIGMA = 3.2
TAIL = 19


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform_residues(g: np.random.Generator, mods, n: int) -> np.ndarray:
    """[len(mods)][n] uint64, limb i uniform in [0, mods[i])."""
    out = np.empty((len(mods), n), dtype=np.uint64)
    for i, q in enumerate(mods):
        out[i] = g.integers(0, int(q), size=n, dtype=np.uint64)
    return out


def binary_poly(g: np.random.Generator, n: int) -> np.ndarray:
    return g.integers(0, 2, size=n, dtype=np.int64)


def gaussian_poly(g: np.random.Generator, n: int, sigma: float = SIGMA) -> np.ndarray:
    return np.clip(np.rint(g.normal(0.0, sigma, size=n)), -TAIL, TAIL).astype(np.int64)


def real_slots(g: np.random.Generator, t: int) -> np.ndarray:
    return g.uniform(-1.0, 1.0, size=t)


def complex_slots(g: np.random.Generator, t: int) -> np.ndarray:
    return g.uniform(-1.0, 1.0, size=t) + 1j * g.uniform(-1.0, 1.0, size=t)


def bag(g: np.random.Generator, m: int, w: int | None = None, zipf_s: float = 1.1):
    """Counted 1-hot bag v (v = sum_i x_i), w tokens, Zipf ids over [0, m)."""
    if w is None:
        w = int(g.integers(50, 601))
    ids = (g.zipf(zipf_s, size=w) - 1) % m
    v = np.bincount(ids, minlength=m).astype(np.float64)
    return v, w


class KeyRandomness:
    """Everything KEYGEN/ENC draw, for a parameter set with L primes + P."""

    def __init__(self, seed: int, log_n: int, q: list[int], P: int):
        self.seed, self.log_n, self.q, self.P = seed, log_n, list(q), P
        self.n = 1 << log_n
        g = rng(seed)
        self.s = binary_poly(g, self.n)
        self.pk_a = uniform_residues(g, self.q, self.n)
        self.pk_e = gaussian_poly(g, self.n)

    def switch_key(self, tag: int, dnum: int | None = None, special: list | None = None):
        """(a [dnum][L+K][N], e [dnum][N]) for one key-switching key; tag distinguishes
        keys.  Defaults: dnum = L digits, one special prime P (alpha = 1)."""
        g = rng(self.seed * 1000003 + 17 + tag)
        L = len(self.q)
        dnum = L if dnum is None else dnum
        ext = self.q + (list(special) if special is not None else [self.P])
        a = np.empty((dnum, len(ext), self.n), dtype=np.uint64)
        for j in range(dnum):
            a[j] = uniform_residues(g, ext, self.n)
        e = np.stack([gaussian_poly(g, self.n) for _ in range(dnum)])
        return a, e

    def enc(self, tag: int):
        """(u, e0, e1) for one encryption."""
        g = rng(self.seed * 7919 + 101 + tag)
        return binary_poly(g, self.n), gaussian_poly(g, self.n), gaussian_poly(g, self.n)
