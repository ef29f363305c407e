"""Pins for the oracle's HMult front-end (tensor product + relinearisation) and Rescale
(§3.6.5; Table 1).

Pins used (none re-types the oracle's own formula):
* Tensor: (d0, d1, d2) decrypts under (1, s, s^2) to the schoolbook negacyclic product m1*m2 of
  the two messages EXACTLY (integer convolution in numpy, independent of every NTT).
* HMult: decryption of the relinearised product is m1*m2 within the KeySwitch noise bound.
* Rescale: closed form of CKKS rescaling -- the CRT value of the output equals round(X / q_l) of
  the CRT value X of the input, coefficient by coefficient (big-int Python); exact division
  X = q_l * Y returns Y; |X| < q_l / 2 returns 0 (reading 15: centered SwitchModulo).
"""
import math

import numpy as np
import pytest

import hks_synth as S
from helpers import Keys, encrypt_under, ks_bound


def negacyclic(a, b):
    """Schoolbook product in Z[X]/(X^N + 1) of small integer polynomials."""
    n = len(a)
    full = np.convolve(np.asarray(a, dtype=np.int64), np.asarray(b, dtype=np.int64))
    out = full[:n].copy()
    out[: n - 1] -= full[n:]
    return out


def crt(residues, primes):
    M = math.prod(primes)
    v = 0
    for r, p in zip(residues, primes):
        Mi = M // p
        v += int(r) * Mi * pow(Mi, -1, p)
    return v % M


def decrypt3(c, d0, d1, d2, s_eval, level):
    """Centered CRT of INTT(d0 + d1 s + d2 s^2) -- decryption of a degree-2 ciphertext."""
    idx = list(range(level + 1))
    s = s_eval[: level + 1]
    s2 = c.mul(s, s, idx)
    t = c.add(d0, c.add(c.mul(d1, s, idx), c.mul(d2, s2, idx), idx), idx)
    return c.crt_centered(c.intt(t, idx), level)


@pytest.mark.parametrize("name,level", [("T10", 4), ("T10", 1), ("T12", 6), ("C1p", 2)])
def test_tensor_decrypts_to_exact_product(orc, name, level):
    cfg = S.config(name)
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg.seed)
    g = S.rng(cfg.seed + 11)
    m1, a0, a1 = encrypt_under(c, g, keys.s_eval, level, 18)
    m2, b0, b1 = encrypt_under(c, g, keys.s_eval, level, 18)
    d0, d1, d2 = c.tensor(a0, a1, b0, b1, level)
    got = decrypt3(c, d0, d1, d2, keys.s_eval, level)
    assert [int(v) for v in negacyclic(m1, m2)] == got


def test_tensor_is_bilinear_not_symmetric_in_halves(orc):
    # swapping the two ciphertexts leaves the tensor unchanged; swapping halves inside one does not
    cfg = S.config("T10")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(5)
    lv = 3
    a0, a1, b0, b1 = (S.uniform_limbs(g, c.q[: lv + 1], c.n) for _ in range(4))
    t1 = c.tensor(a0, a1, b0, b1, lv)
    t2 = c.tensor(b0, b1, a0, a1, lv)
    t3 = c.tensor(a1, a0, b0, b1, lv)
    assert all((x == y).all() for x, y in zip(t1, t2))
    assert not (t1[0] == t3[0]).all() and not (t1[2] == t3[2]).all()


@pytest.mark.parametrize("name,levels", [("T10", [4, 3, 1, 0]), ("T12", [6, 2]), ("C1p", [2, 0])])
def test_hmult_decrypts_within_ks_bound(orc, name, levels):
    cfg = S.config(name)
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg.seed)
    evk = keys.relin()
    g = S.rng(cfg.seed + 12)
    for level in levels:
        m1, a0, a1 = encrypt_under(c, g, keys.s_eval, level, 14)
        m2, b0, b1 = encrypt_under(c, g, keys.s_eval, level, 14)
        o0, o1 = c.hmult(a0, a1, b0, b1, evk, level)
        dec = c.crt_centered(c.decrypt_coeff(o0, o1, keys.s_eval, level), level)
        want = negacyclic(m1, m2)
        bound = ks_bound(c, level, keys.B_e, keys.h)
        Q = math.prod(c.q[: level + 1])
        assert bound + 2 ** 40 < Q // 2
        err = max(abs(int(a) - int(b)) for a, b in zip(dec, want))
        assert err <= bound, (err, bound)


# ------------------------------------------------------------------ Rescale

def rescale_coeff(c, res_coef, level):
    """Oracle rescale driven from COEFF residues (NTT pinned separately): returns COEFF residues."""
    idx = list(range(level + 1))
    out = c.rescale(c.ntt(np.ascontiguousarray(res_coef, dtype=np.uint64), idx), level)
    return c.intt(out, list(range(level)))


@pytest.mark.parametrize("name,level", [("T10", 4), ("T10", 1), ("T12", 6), ("T12", 3), ("C1", 2)])
def test_rescale_is_rounded_division(orc, name, level):
    cfg = S.config(name)
    c = orc.Ctx.from_config(cfg)
    g = S.rng(cfg.seed + 13)
    qs = c.q[: level + 1]
    ql = qs[-1]
    Qp = math.prod(qs[:-1])
    res = S.uniform_limbs(g, qs, c.n)                 # uniform residues = uniform X in [0, Q)
    out = rescale_coeff(c, res, level)
    for k in range(0, c.n, max(1, c.n // 96)):
        X = crt([res[i][k] for i in range(level + 1)], qs)
        Y = crt([out[i][k] for i in range(level)], qs[:-1])
        assert Y == ((2 * X + ql) // (2 * ql)) % Qp, k     # round(X / q_l), q_l odd: no ties


def test_rescale_exact_division_and_small_values(orc):
    cfg = S.config("T12")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(3)
    level = 5
    qs = c.q[: level + 1]
    ql = qs[-1]
    # X = q_l * Y for signed Y of 100 bits -> Y exactly
    Y = [int(v) for v in g.integers(-(1 << 50), 1 << 50, size=c.n)]
    Y = [y * (1 << 50) + int(g.integers(0, 1 << 50)) for y in Y]
    res = np.array([[(ql * y) % q for y in Y] for q in qs], dtype=np.uint64)
    out = rescale_coeff(c, res, level)
    want = np.array([[y % q for y in Y] for q in qs[:-1]], dtype=np.uint64)
    assert (out == want).all()
    # |X| < q_l / 2 -> 0; X = +-(q_l - 1)/2 are the extreme values that still round to 0
    h = (ql - 1) // 2
    X = [int(v) for v in g.integers(-(1 << 58), 1 << 58, size=c.n)]
    X[0], X[1] = h, -h
    res = np.array([[x % q for x in X] for q in qs], dtype=np.uint64)
    assert (rescale_coeff(c, res, level) == 0).all()
    # X = (q_l + 1) / 2 rounds up to 1, X = -(q_l + 1) / 2 rounds to -1
    X = [0] * c.n
    X[0], X[1] = h + 1, -(h + 1)
    res = np.array([[x % q for x in X] for q in qs], dtype=np.uint64)
    out = rescale_coeff(c, res, level)
    assert [int(out[i][0]) for i in range(level)] == [1] * level
    assert [int(out[i][1]) for i in range(level)] == [q - 1 for q in qs[:-1]]
