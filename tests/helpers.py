"""Shared test helpers: host/device conversion and seeded key/ciphertext material.

Keys and ciphertexts for parity tests come from the oracle's client-side functions (real keys,
SURVEY.md §8(c) oracle-side keygen); the random numbers come from hks_synth."""
import math

import numpy as np

import hks_synth as S


def to_dev(a: np.ndarray, device="cuda:0"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(device)


def to_host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def empty_dev(shape, device="cuda:0"):
    import torch
    return torch.empty(shape, dtype=torch.int64, device=device)


class Keys:
    def __init__(self, c, seed):
        g = S.rng(seed)
        self.c, self.g = c, g
        self.s = S.ternary(g, c.n)
        self.h = int(np.count_nonzero(self.s))
        self.s_eval = c.secret_eval(self.s)
        self.nk = c.nq + c.np
        self.B_e = 0

    def ksk(self, s_old_eval):
        c, g = self.c, self.g
        a = np.stack([S.uniform_limbs(g, c.primes, c.n) for _ in range(c.dnum)])
        e = np.stack([S.gaussian(g, c.n) for _ in range(c.dnum)])
        self.B_e = max(self.B_e, int(np.abs(e).max()))
        return c.keygen_ks(self.s_eval, s_old_eval, a, e)

    def relin(self):
        idx = list(range(self.nk))
        return self.ksk(self.c.mul(self.s_eval, self.s_eval, idx))

    def rot(self, k):
        return self.ksk(self.c.automorph(self.s_eval, k))


def ks_bound(c, level, B_e, h):
    P = math.prod(c.p)
    tot = 0
    for lo, hi in c.digits(level):
        tot += c.n * (hi - lo) * math.prod(c.q[lo:hi]) * B_e
    return -(-tot // P) + (c.np + 1) * (1 + h)


def encrypt_under(c, g, s_old_eval, level, mbits):
    qidx = list(range(level + 1))
    m = g.integers(-(1 << mbits), 1 << mbits, size=c.n, dtype=np.int64)
    c1 = S.uniform_limbs(g, c.q[: level + 1], c.n)
    mev = c.ntt(c.lift(m, qidx), qidx)
    c0 = c.sub(mev, c.mul(c1, s_old_eval[: level + 1], qidx), qidx)
    return m, c0, c1
