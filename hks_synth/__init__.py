"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no NTT, no base conversion, no
key switching, no modular products).  It only draws numbers:

* NTT-friendly prime chains (SURVEY.md §8(c) reading 6: P = the K largest primes
  < 2^B with p = 1 mod 2N, Q = the next L+1 below them);
* uniform residues per limb, ternary secrets, rounded-Gaussian errors
  (sigma = 3.19), all from numpy PCG64(seed);
* the five workload configurations of BASELINE.json.

Randomness the method consumes (the key's `a`, the errors `e`, the secret `s`)
is drawn here and passed in to both the oracle and the CUDA path.
"""
from __future__ import annotations

import dataclasses
import functools

import numpy as np

__all__ = [
    "is_prime", "ntt_primes", "Config", "config", "rng", "uniform_limbs",
    "ternary", "gaussian", "galois_rot", "GALOIS_CONJ",
]

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (fixed witness set)."""
    if n < 2:
        return False
    for b in _MR_BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
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


@functools.lru_cache(maxsize=None)
def ntt_primes(log_n: int, count: int, bits: int) -> tuple:
    """The `count` largest primes p < 2^bits with p = 1 (mod 2N), descending."""
    step = 2 << log_n
    cand = ((1 << bits) - 1) // step * step + 1
    if cand >= (1 << bits):
        cand -= step
    out = []
    while len(out) < count:
        if cand < step:
            raise ValueError("prime exhaustion")
        if is_prime(cand):
            out.append(cand)
        cand -= step
    return tuple(out)


@dataclasses.dataclass(frozen=True)
class Config:
    """A workload from BASELINE.json `configs` (recipe in SURVEY.md §8(d))."""
    name: str
    log_n: int
    q: tuple          # L+1 chain primes
    p: tuple          # K special primes
    dnum: int
    level: int        # level the headline op runs at
    seed: int

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def L(self) -> int:
        return len(self.q) - 1

    @property
    def K(self) -> int:
        return len(self.p)

    @property
    def alpha(self) -> int:
        return -(-(self.L + 1) // self.dnum)

    def beta(self, level: int) -> int:
        return -(-(level + 1) // self.alpha)

    @property
    def bits(self) -> int:
        return max(max(self.q), max(self.p)).bit_length()


def _mk(name, log_n, nq, np_, dnum, bits, seed, level=None):
    primes = ntt_primes(log_n, nq + np_, bits)
    p = primes[:np_]
    q = primes[np_:np_ + nq]
    return Config(name, log_n, tuple(q), tuple(p), dnum,
                  nq - 1 if level is None else level, seed)


def config(name: str) -> Config:
    """C1, C1p (C1 with dnum=3), C2, C4, and small test shapes.

    C1  = N=2^12, 3 Q + 1 P < 2^50, dnum=1          (BASELINE.json configs[0])
    C2  = N=2^16, L=29, K=10, 60-bit, dnum=3        (configs[1], the bench workload)
    C3  = C2 parameters, 8 ct x 8 hoisted rotations (configs[2])
    C4  = N=2^17, L=35, K=9, 60-bit, dnum=4         (configs[3])
    C5  = C2 parameters, BOOT_SHAPE v1              (configs[4])
    """
    table = {
        "C1": lambda: _mk("C1", 12, 3, 1, 1, 50, 1001),
        "C1p": lambda: _mk("C1p", 12, 3, 1, 3, 50, 1001),
        "C2": lambda: _mk("C2", 16, 30, 10, 3, 60, 1002),
        "C3": lambda: _mk("C3", 16, 30, 10, 3, 60, 1003),
        "C4": lambda: _mk("C4", 17, 36, 9, 4, 60, 1004),
        "C5": lambda: _mk("C5", 16, 30, 10, 3, 60, 1005),
        # small shapes for CPU/GPU parity sweeps: several tiles, ragged digits
        "T10": lambda: _mk("T10", 10, 5, 2, 3, 60, 2010),      # alpha=2, digits [2,2,1]
        "T12": lambda: _mk("T12", 12, 7, 3, 3, 60, 2012),      # alpha=3, digits [3,3,1]
        "T13": lambda: _mk("T13", 13, 6, 2, 3, 59, 2013),
        "T14": lambda: _mk("T14", 14, 8, 3, 3, 60, 2014),
        "T16s": lambda: _mk("T16s", 16, 6, 2, 3, 60, 2016),    # full N=2^16, few limbs
        "T17s": lambda: _mk("T17s", 17, 5, 2, 3, 60, 2017),    # full N=2^17, few limbs
    }
    return table[name]()


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform_limbs(g: np.random.Generator, primes, n: int) -> np.ndarray:
    """[len(primes)][n] uint64, limb b uniform in [0, primes[b])."""
    out = np.empty((len(primes), n), dtype=np.uint64)
    for b, q in enumerate(primes):
        out[b] = g.integers(0, q, size=n, dtype=np.uint64)
    return out


def ternary(g: np.random.Generator, n: int) -> np.ndarray:
    """Uniform ternary secret coefficients in {-1, 0, 1} (SURVEY.md §8(c) keygen)."""
    return g.integers(-1, 2, size=n, dtype=np.int64)


def gaussian(g: np.random.Generator, n: int, sigma: float = 3.19) -> np.ndarray:
    """Rounded Gaussian (round half away from zero), sigma = 3.19."""
    x = g.normal(0.0, sigma, size=n)
    return (np.sign(x) * np.floor(np.abs(x) + 0.5)).astype(np.int64)


def galois_rot(r: int, log_n: int) -> int:
    """Galois element 5^r mod 2N for a slot rotation by r."""
    return pow(5, r, 2 << log_n)


def GALOIS_CONJ(log_n: int) -> int:
    """Conjugation element 2N-1."""
    return (2 << log_n) - 1
