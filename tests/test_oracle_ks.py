"""Pins for the oracle's base conversion, ModUp, key inner product, ModDown, KeySwitch and
hoisted rotations (SURVEY.md §8(c) "What pins each part").

Pins used (none re-types the oracle's own formula):
* BConv / ModUp: big-int CRT overshoot invariant out = X + u*Q' with one u in [0, #src)
  shared by all targets.
* ModDown: ModDown(P*y) = y exactly; ModDown(P*y + a) = y + ModDown(a); big-int
  ModDown(a) = floor(A/P) - v with v in [0, K).
* Key inner product: special keys (unit / zero digits) and the automorphism commuting rule.
* KeySwitch / relinearisation / rotation / hoisted rotation: decryption of the result is
  the expected message within the analytic noise bound (SURVEY.md §8(c) "decryption bound").
* Structural goldens: digit partition, K, key sizes, transform count.
"""
import math

import numpy as np
import pytest

import hks_synth as S
from conftest import read_golden


def crt(residues, primes):
    """Big-int CRT of one coefficient's residues -> value in [0, prod(primes))."""
    M = math.prod(primes)
    v = 0
    for r, p in zip(residues, primes):
        Mi = M // p
        v += int(r) * Mi * pow(Mi, -1, p)
    return v % M


def find_u(out_res, X, Qs, tgt_primes, umax):
    us = [u for u in range(umax) if all((X + u * Qs) % t == int(o) for o, t in zip(out_res, tgt_primes))]
    return us


# ------------------------------------------------------------------ structure goldens

def test_digits_golden(orc):
    for L, dnum, level, alpha, sizes in read_golden("digits.txt"):
        L, dnum, level, alpha = int(L), int(dnum), int(level), int(alpha)
        q = S.ntt_primes(4, L + 1 + 1, 40)
        c = orc.Ctx(4, q[1:], q[:1], dnum)
        assert c.alpha == alpha == -(-(L + 1) // dnum)
        assert [hi - lo for lo, hi in c.digits(level)] == [int(s) for s in sizes.split(",")]


def test_ksk_size_golden():
    for log_n, L, dnum, mib in read_golden("ksk_sizes.txt"):
        log_n, L, dnum = int(log_n), int(L), int(dnum)
        K = -(-(L + 1) // dnum)
        nbytes = dnum * 2 * (L + 1 + K) * (1 << log_n) * 8     # evk layout [dnum][2][L+1+K][N] u64
        assert nbytes == int(mib) * 2 ** 20
        # neighbouring K would not reproduce the printed size
        assert dnum * 2 * (L + 1 + K + 1) * (1 << log_n) * 8 != int(mib) * 2 ** 20


def test_transform_count_golden(orc):
    for L, dnum, level, approx, tol in read_golden("transform_counts.txt"):
        L, dnum, level = int(L), int(dnum), int(level)
        q = S.ntt_primes(4, L + 1 + 8, 40)
        c = orc.Ctx(4, q[8:], q[:8], dnum)
        beta = c.beta(level)
        count = (level + 1) + beta * (level + 1 + c.np) - (level + 1)
        assert abs(count - float(approx)) <= float(tol) * float(approx)


# ------------------------------------------------------------------ BConv / ModUp

def test_bconv_crt_overshoot(orc):
    cfg = S.config("T12")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(21)
    src, dst = [0, 1, 2], [3, 4, 5, 6, 7, 8, 9]
    sp = [c.primes[i] for i in src]
    tp = [c.primes[i] for i in dst]
    x = S.uniform_limbs(g, sp, c.n)
    out = c.bconv(x, src, dst)
    Qs = math.prod(sp)
    seen_u = set()
    for n in list(range(0, c.n, 37)) + [c.n - 1]:
        X = crt(x[:, n], sp)
        us = find_u(out[:, n], X, Qs, tp, len(src))
        assert len(us) == 1, n
        seen_u.add(us[0])
    assert seen_u <= set(range(len(src))) and len(seen_u) > 1
    # zero -> zero; a single-limb source is an exact lift (u = 0): out = x mod t
    assert (c.bconv(np.zeros_like(x), src, dst) == 0).all()
    one = c.bconv(x[:1], src[:1], dst)
    for t, p in enumerate(tp):
        assert (one[t] == x[0] % np.uint64(p)).all()


@pytest.mark.parametrize("level", [6, 3, 0])
def test_modup_invariant(orc, level):
    cfg = S.config("T12")      # L=6, dnum=3 -> alpha=3, digits [3,3,1] at level 6, K=3
    c = orc.Ctx.from_config(cfg)
    g = S.rng(22 + level)
    qidx = list(range(level + 1))
    d = S.uniform_limbs(g, c.q[: level + 1], c.n)
    ext = c.modup(d, level)
    eidx = c.ext_primes(level)
    ep = [c.primes[i] for i in eidx]
    dco = c.intt(d, qidx)
    assert ext.shape[0] == c.beta(level)
    for j, (lo, hi) in enumerate(c.digits(level)):
        assert (ext[j, lo:hi] == d[lo:hi]).all()              # own-digit limbs pass through in EVAL
        Dco = c.intt(ext[j], eidx)
        Qj = math.prod(c.q[lo:hi])
        for n in range(0, c.n, 97):
            X = crt(dco[lo:hi, n], c.q[lo:hi])
            us = find_u(Dco[:, n], X, Qj, ep, hi - lo)
            assert len(us) == 1


# ------------------------------------------------------------------ key inner product

def test_kip_special_keys(orc):
    cfg = S.config("T12")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(23)
    level = 6
    nk = c.nq + c.np
    ne = level + 1 + c.np
    ext = np.stack([S.uniform_limbs(g, [c.primes[i] for i in c.ext_primes(level)], c.n)
                    for _ in range(c.beta(level))])
    evk = np.zeros((c.dnum, 2, nk, c.n), np.uint64)
    evk[1, 0] = 1                  # b_1 = 1, every other b_j = 0  -> acc0 = D_1
    evk[:, 1] = 1                  # a_j = 1 for all j             -> acc1 = sum_j D_j
    acc = c.kip(ext, evk, level)
    assert (acc[0] == ext[1]).all()
    eidx = c.ext_primes(level)
    s = ext[0]
    for j in range(1, c.beta(level)):
        s = c.add(s, ext[j], eidx)
    assert (acc[1] == s).all()
    # galois: kip(ext, evk, k) == kip(pi_k(ext), evk, 1)
    evk = S.uniform_limbs(g, list(c.primes) * (2 * c.dnum), c.n).reshape(c.dnum, 2, nk, c.n)
    k = S.galois_rot(3, cfg.log_n)
    rot = np.stack([c.automorph(ext[j], k) for j in range(ext.shape[0])])
    assert (c.kip(ext, evk, level, k) == c.kip(rot, evk, level, 1)).all()
    assert acc.shape == (2, ne, c.n)


# ------------------------------------------------------------------ ModDown

def test_moddown_exact_identities(orc):
    cfg = S.config("T12")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(24)
    for level in (6, 2, 0):
        qidx = list(range(level + 1))
        eidx = c.ext_primes(level)
        P = math.prod(c.p)
        y = S.uniform_limbs(g, c.q[: level + 1], c.n)
        Pq = np.array([[P % q] * c.n for q in c.q[: level + 1]], dtype=np.uint64)
        acc = np.zeros((len(eidx), c.n), np.uint64)
        acc[: level + 1] = c.mul(y, Pq, qidx)
        assert (c.moddown(acc, level) == y).all()               # ModDown(P*y) = y exactly
        a = S.uniform_limbs(g, [c.primes[i] for i in eidx], c.n)
        acc2 = a.copy()
        acc2[: level + 1] = c.add(acc[: level + 1], a[: level + 1], qidx)
        assert (c.moddown(acc2, level) == c.add(y, c.moddown(a, level), qidx)).all()


def test_moddown_bigint_floor(orc):
    cfg = S.config("T12")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(25)
    level = 5
    eidx = c.ext_primes(level)
    ep = [c.primes[i] for i in eidx]
    a = S.uniform_limbs(g, ep, c.n)
    out = c.moddown(a, level)
    aco = c.intt(a, eidx)
    oco = c.intt(out, list(range(level + 1)))
    P = math.prod(c.p)
    Q = math.prod(c.q[: level + 1])
    vs = set()
    for n in range(0, c.n, 53):
        A = crt(aco[:, n], ep)
        R = crt(oco[:, n], c.q[: level + 1])
        v = (A // P - R) % Q
        assert 0 <= v < c.np
        vs.add(v)
    assert len(vs) > 1


# ------------------------------------------------------------------ end-to-end: decryption bound

def ks_bound(c, level, B_e, h):
    P = math.prod(c.p)
    tot = 0
    for lo, hi in c.digits(level):
        Qj = math.prod(c.q[lo:hi])
        tot += c.n * (hi - lo) * Qj * B_e
    return -(-tot // P) + (c.np + 1) * (1 + h)


def automorph_int(m, k, n):
    out = [0] * n
    for i, v in enumerate(m):
        e = i * k % (2 * n)
        if e >= n:
            out[e - n] -= v
        else:
            out[e] += v
    return out


class Keys:
    def __init__(self, c, cfg, seed):
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


def encrypt_under(c, g, s_old_eval, level, mbits):
    """c1 uniform over Q_l (EVAL); c0 = m - c1*s_old; m random with |m_i| < 2^mbits."""
    qidx = list(range(level + 1))
    m = g.integers(-(1 << mbits), 1 << mbits, size=c.n, dtype=np.int64) if mbits < 62 else None
    c1 = S.uniform_limbs(g, c.q[: level + 1], c.n)
    mev = c.ntt(c.lift(m, qidx), qidx)
    c0 = c.sub(mev, c.mul(c1, s_old_eval[: level + 1], qidx), qidx)
    return m, c0, c1


def check_decrypt(c, keys, out0, out1, level, expect, bound):
    dec = c.crt_centered(c.decrypt_coeff(out0, out1, keys.s_eval, level), level)
    err = max(abs(int(a) - int(b)) for a, b in zip(dec, expect))
    assert err <= bound, (err, bound)
    return err


@pytest.mark.parametrize("name,levels", [("C1", [2]), ("C1p", [2, 1, 0]), ("T12", [6, 5, 2, 0]),
                                         ("T10", [4, 3])])
def test_keyswitch_relin_decrypts(orc, name, levels):
    cfg = S.config(name)
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg, cfg.seed)
    evk = keys.relin()
    s2 = c.mul(keys.s_eval, keys.s_eval, list(range(keys.nk)))
    g = S.rng(cfg.seed + 1)
    for level in levels:
        m, c0, c1 = encrypt_under(c, g, s2, level, 20)
        o0, o1 = c.keyswitch(c0, c1, evk, level)
        bound = ks_bound(c, level, keys.B_e, keys.h)
        Q = math.prod(c.q[: level + 1])
        assert bound < Q // 4, "bound must be meaningful"
        check_decrypt(c, keys, o0, o1, level, list(m), bound)


def test_keyswitch_c1_large_message(orc):
    # C1: P (one ~2^50 prime) < Q_0: noise ~ 2^117; check with |m| < 2^60 (SURVEY.md reading 17)
    cfg = S.config("C1")
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg, 77)
    evk = keys.relin()
    s2 = c.mul(keys.s_eval, keys.s_eval, list(range(keys.nk)))
    g = S.rng(78)
    m, c0, c1 = encrypt_under(c, g, s2, 2, 60)
    o0, o1 = c.keyswitch(c0, c1, evk, 2)
    bound = ks_bound(c, 2, keys.B_e, keys.h)
    assert 2 ** 100 < bound < math.prod(c.q) // 4
    check_decrypt(c, keys, o0, o1, 2, list(m), bound)


def test_keyswitch_zero_and_linear(orc):
    cfg = S.config("T10")
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg, 5)
    evk = keys.relin()
    level = 4
    z = np.zeros((level + 1, c.n), np.uint64)
    o0, o1 = c.keyswitch(z, z, evk, level)
    assert (o0 == 0).all() and (o1 == 0).all()                  # d = 0 -> zero pair


def test_rotation_and_hoisted(orc):
    cfg = S.config("T12")
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg, 31)
    ks = [S.galois_rot(r, cfg.log_n) for r in (1, 2, 5)] + [S.GALOIS_CONJ(cfg.log_n)]
    evks = [keys.rot(k) for k in ks]
    g = S.rng(32)
    level = 6
    m, c0, c1 = encrypt_under(c, g, keys.s_eval, level, 20)    # fresh ct under s
    bound = ks_bound(c, level, keys.B_e, keys.h)
    h0, h1 = c.rotate_hoisted(c0, c1, evks, level, ks)
    any_diff = False
    for k, evk, a0, a1 in zip(ks, evks, h0, h1):
        want = automorph_int(list(m), k, c.n)
        check_decrypt(c, keys, a0, a1, level, want, bound)          # hoisted decrypts to pi_k(m)
        u0, u1 = c.rotate(c0, c1, evk, level, k)
        check_decrypt(c, keys, u0, u1, level, want, bound)          # unhoisted too
        any_diff |= bool((u1 != a1).any())
    assert any_diff      # reading 14: hoisted is decrypt-equal, not bit-equal, to unhoisted
    # one rotation through the hoisted path == the same rotation alone through it
    s0, s1 = c.rotate_hoisted(c0, c1, evks[1:2], level, ks[1:2])
    assert (s0[0] == h0[1]).all() and (s1[0] == h1[1]).all()


@pytest.mark.slow
def test_keyswitch_c2_decrypts(orc):
    cfg = S.config("C2")
    c = orc.Ctx.from_config(cfg)
    keys = Keys(c, cfg, cfg.seed)
    evk = keys.relin()
    s2 = c.mul(keys.s_eval, keys.s_eval, list(range(keys.nk)))
    g = S.rng(cfg.seed + 1)
    level = 29
    m, c0, c1 = encrypt_under(c, g, s2, level, 20)
    o0, o1 = c.keyswitch(c0, c1, evk, level)
    bound = ks_bound(c, level, keys.B_e, keys.h)
    assert bound < 2 ** 26
    check_decrypt(c, keys, o0, o1, level, list(m), bound)
