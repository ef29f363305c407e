"""Pins for the oracle's fused plaintext-weighted sum and BSGS linear transform (SURVEY.md §8(f)
NEXT-2; PAPER.md:352 weighted-sum fusion, §3.6.7 BSGS with hoisted rotations;
SPEC.md:576-583).

Pins used (none re-types the oracle's own formula):
* Weighted sum: sum_j p_j * (x0_j, x1_j) decrypts EXACTLY to the schoolbook sum_j p_j * m_j.
* Linear transform: decryption equals the integer-ring BSGS result
  sum_i sigma_{g_i}( sum_j p_ij * sigma_{b_j}(m) ) (numpy convolutions + signed coefficient
  automorphisms, no NTT) within the propagated KeySwitch noise bound; the identity transform
  (n1 = n2 = 1, p = 1) returns the input ciphertext bit for bit.
"""
import math

import numpy as np
import pytest

import hks_synth as S
from helpers import Keys, encrypt_under, ks_bound


def negacyclic(a, b):
    n = len(a)
    full = np.convolve(np.asarray(a, dtype=np.int64), np.asarray(b, dtype=np.int64))
    out = full[:n].copy()
    out[: n - 1] -= full[n:]
    return out


def sigma(m, k):
    """X -> X^k on an integer polynomial mod X^N + 1."""
    n = len(m)
    out = np.zeros(n, dtype=np.int64)
    for i, v in enumerate(m):
        e = i * k % (2 * n)
        if e >= n:
            out[e - n] -= v
        else:
            out[e] += v
    return out


def small_poly(g, n, lim=2):
    return g.integers(-lim, lim + 1, size=n, dtype=np.int64)


def to_eval(c, poly, level):
    idx = list(range(level + 1))
    return c.ntt(c.lift(poly, idx), idx)


def test_pt_wsum_decrypts_exactly(orc):
    cfg = S.config("T10")
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, 31)
    g = S.rng(32)
    level = 3
    ms, x0, x1, ps = [], [], [], []
    for _ in range(5):
        m, a0, a1 = encrypt_under(c, g, keys.s_eval, level, 12)
        ms.append(m), x0.append(a0), x1.append(a1)
        ps.append(small_poly(g, c.n, 3))
    o0, o1 = c.pt_wsum([to_eval(c, p, level) for p in ps], x0, x1, level)
    dec = c.crt_centered(c.decrypt_coeff(o0, o1, keys.s_eval, level), level)
    want = sum(negacyclic(p, m) for p, m in zip(ps, ms))
    assert [int(v) for v in want] == dec


def test_lintrans_identity_is_exact(orc):
    cfg = S.config("T12")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(33)
    level = 4
    c0, c1 = (S.uniform_limbs(g, c.q[: level + 1], c.n) for _ in range(2))
    one = to_eval(c, np.eye(1, c.n, dtype=np.int64)[0], level)
    o0, o1 = c.lintrans(c0, c1, level, 1, 1, [], [], [], [], [one])
    assert (o0 == c0).all() and (o1 == c1).all()


@pytest.mark.parametrize("name,level,n1,n2", [("T12", 6, 3, 3), ("T12", 4, 4, 1), ("T12", 5, 1, 3), ("T10", 4, 2, 2)])
def test_lintrans_decrypts_to_bsgs_ring_result(orc, name, level, n1, n2):
    cfg = S.config(name)
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg.seed + 3)
    g = S.rng(cfg.seed + 4)
    bgal = [S.galois_rot(j, cfg.log_n) for j in range(1, n1)]
    ggal = [S.galois_rot(i * n1, cfg.log_n) for i in range(1, n2)]
    bk = [keys.rot(k) for k in bgal]
    gk = [keys.rot(k) for k in ggal]
    m, c0, c1 = encrypt_under(c, g, keys.s_eval, level, 10)
    ps = [small_poly(g, c.n) for _ in range(n1 * n2)]
    o0, o1 = c.lintrans(c0, c1, level, n1, n2, bgal, bk, ggal, gk, [to_eval(c, p, level) for p in ps])
    babies = [m] + [sigma(m, k) for k in bgal]
    want = np.zeros(c.n, dtype=np.int64)
    for i in range(n2):
        inner = sum(negacyclic(ps[i * n1 + j], babies[j]) for j in range(n1))
        want += inner if i == 0 else sigma(inner, ggal[i - 1])
    dec = c.crt_centered(c.decrypt_coeff(o0, o1, keys.s_eval, level), level)
    B = ks_bound(c, level, keys.B_e, keys.h)
    l1 = [int(np.abs(p).sum()) for p in ps]
    bound = sum(sum(l1[i * n1 + j] * B for j in range(1, n1)) + (B if i else 0) for i in range(n2))
    assert bound < math.prod(c.q[: level + 1]) // 4
    err = max(abs(int(a) - int(b)) for a, b in zip(dec, want))
    assert err <= bound, (err, bound)
    if n1 > 1 or n2 > 1:
        assert err > 0          # sanity: the key switches add noise
