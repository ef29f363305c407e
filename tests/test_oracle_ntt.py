"""Pins for the oracle's modular arithmetic, psi and NTT/INTT (SURVEY.md §8(c) "What pins each part").

Every check compares the oracle with something other than itself: hand arithmetic,
brute force over tiny fields, the schoolbook negacyclic product, algebraic identities.
"""
import numpy as np
import pytest

import hks_synth as S
from conftest import read_golden


def schoolbook_negacyclic(a, b, p):
    """O(N^2) product in Z_p[X]/(X^N+1) with Python ints."""
    n = len(a)
    out = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            v = int(a[i]) * int(b[j])
            if k >= n:
                out[k - n] -= v
            else:
                out[k] += v
    return [x % p for x in out]


def small_ctx(orc, log_n, count=2, bits=30):
    primes = S.ntt_primes(log_n, count + 1, bits)
    return orc.Ctx(log_n, primes[1:], primes[:1], 1)


def test_modarith_golden(orc):
    c = orc.Ctx(3, [17], [97], 1)   # 17 = 1 mod 16, 97 = 1 mod 16
    for op, a, b, p, want in read_golden("modarith.txt"):
        assert int(p) == 17
        A = np.full((1, 8), int(a), dtype=np.uint64)
        B = np.full((1, 8), int(b), dtype=np.uint64)
        got = getattr(c, op)(A, B, [0])
        assert (got == int(want)).all(), (op, a, b)


def test_modarith_exhaustive_small_prime(orc):
    # exhaustive over Z_17 x Z_17 vs Python's exact integer arithmetic
    c = orc.Ctx(3, [17], [97], 1)
    a = np.repeat(np.arange(17, dtype=np.uint64), 17)
    b = np.tile(np.arange(17, dtype=np.uint64), 17)
    pad = (-len(a)) % 8
    a = np.concatenate([a, np.zeros(pad, np.uint64)]).reshape(-1, 8)
    b = np.concatenate([b, np.zeros(pad, np.uint64)]).reshape(-1, 8)
    idx = [0] * a.shape[0]
    for op, f in (("add", lambda x, y: (x + y) % 17), ("sub", lambda x, y: (x - y) % 17),
                  ("mul", lambda x, y: x * y % 17)):
        got = getattr(c, op)(a, b, idx).ravel()
        want = [f(int(x), int(y)) for x, y in zip(a.ravel(), b.ravel())]
        assert list(map(int, got)) == want


def test_modarith_random_60bit(orc):
    cfg = S.config("T10")
    c = orc.Ctx.from_config(cfg)
    g = S.rng(7)
    q = cfg.q[0]
    a = S.uniform_limbs(g, [q] * 64, c.n)
    b = S.uniform_limbs(g, [q] * 64, c.n)
    got = c.mul(a, b, [0] * 64)
    sel = g.integers(0, a.size, 20000)
    af, bf, gf = a.ravel(), b.ravel(), got.ravel()
    for i in sel:
        assert int(gf[i]) == int(af[i]) * int(bf[i]) % q


def test_primality(orc):
    assert orc.is_prime(97) and orc.is_prime((1 << 61) - 1)
    assert not orc.is_prime(561) and not orc.is_prime(3215031751)   # Carmichael / strong pseudoprime to 2,3,5,7
    for p in S.ntt_primes(16, 5, 60):
        assert orc.is_prime(p)
    # agreement with trial division on a dense small range
    for x in range(2, 3000):
        assert orc.is_prime(x) == all(x % d for d in range(2, int(x ** 0.5) + 1))


@pytest.mark.parametrize("p,n", [(17, 8), (97, 16), (193, 32), (257, 64), (7681, 256)])
def test_min_psi_brute_force(orc, p, n):
    # reading 1: psi = minimal x with x^N = -1 (mod p); brute force over all of Z_p
    want = next(x for x in range(2, p) if pow(x, n, p) == p - 1)
    assert orc.min_psi(p, n) == want


def test_min_psi_60bit_properties(orc):
    for log_n in (12, 16, 17):
        for p in S.ntt_primes(log_n, 3, 60):
            n = 1 << log_n
            psi = orc.min_psi(p, n)
            assert pow(psi, n, p) == p - 1 and pow(psi, 2 * n, p) == 1
            # no smaller primitive 2N-th root: every root is psi^k (k odd); check a window of them
            g2 = psi * psi % p
            r = psi
            for _ in range(min(n, 4096)):
                assert r >= psi
                r = r * g2 % p


@pytest.mark.parametrize("log_n", [1, 2, 3, 4, 5, 6])
def test_ntt_convolution_theorem(orc, log_n):
    # pointwise product in EVAL == schoolbook negacyclic product
    c = small_ctx(orc, log_n, count=2, bits=30)
    g = S.rng(100 + log_n)
    for pidx in range(3):
        p = c.primes[pidx]
        a = S.uniform_limbs(g, [p], c.n)
        b = S.uniform_limbs(g, [p], c.n)
        prod = c.intt(c.mul(c.ntt(a, [pidx]), c.ntt(b, [pidx]), [pidx]), [pidx])
        assert list(map(int, prod[0])) == schoolbook_negacyclic(a[0], b[0], p)


def test_ntt_eval_points_and_order(orc):
    # NTT(X)[j] are the N roots of X^N+1, each exactly once; NTT(X)[0] = psi (reading 1);
    # bit-reversed order (reading 2): adjacent outputs are negatives (2brv(2j+1)+1 = 2brv(2j)+1+N).
    for log_n in (4, 8, 10):
        c = small_ctx(orc, log_n, count=1, bits=40)
        p, n = c.primes[0], c.n
        x = np.zeros((1, n), np.uint64)
        x[0, 1] = 1
        ev = [int(v) for v in c.ntt(x, [0])[0]]
        assert ev[0] == c.psi(0)
        assert len(set(ev)) == n and all(pow(v, n, p) == p - 1 for v in ev)
        for j in range(0, n, 2):
            assert (ev[j] + ev[j + 1]) % p == 0
        # the second half of the natural-order roots list (psi^(2k+1), k >= N/2) lands on odd j:
        # brv(j) >= N/2 <=> j odd.
        roots = [pow(c.psi(0), 2 * k + 1, p) for k in range(n)]
        pos = {v: j for j, v in enumerate(ev)}
        for k in range(n):
            assert (pos[roots[k]] % 2 == 1) == (k >= n // 2)


@pytest.mark.parametrize("log_n", [4, 7, 10])
def test_ntt_matches_definition(orc, log_n):
    # against the O(N^2) definition (Horner evaluation at psi^(2brv(j)+1)), all outputs
    cfg = S.config("T10")
    c = orc.Ctx(log_n, S.ntt_primes(log_n, 3, 60)[1:], S.ntt_primes(log_n, 3, 60)[:1], 1)
    g = S.rng(200 + log_n)
    for pidx in range(3):
        a = S.uniform_limbs(g, [c.primes[pidx]], c.n)
        ev = c.ntt(a, [pidx])[0]
        assert (c.ntt_def(a[0], pidx, range(c.n)) == ev).all()
    del cfg


def test_ntt_identities(orc):
    c = small_ctx(orc, 10, count=3, bits=60)
    g = S.rng(11)
    idx = list(range(4))
    a = S.uniform_limbs(g, c.primes, c.n)
    b = S.uniform_limbs(g, c.primes, c.n)
    A, B = c.ntt(a, idx), c.ntt(b, idx)
    assert (c.intt(A, idx) == a).all()                       # INTT o NTT = id
    assert (c.ntt(c.intt(a, idx), idx) == a).all()           # NTT o INTT = id
    assert (c.ntt(c.add(a, b, idx), idx) == c.add(A, B, idx)).all()   # linearity
    const = np.zeros_like(a)
    const[:, 0] = 12345
    assert (c.ntt(const, idx) == 12345).all()                # constant -> constant
    half = np.zeros_like(a)
    half[:, c.n // 2] = 1
    H = c.ntt(half, idx)
    sq = c.intt(c.mul(H, H, idx), idx)                       # (X^{N/2})^2 = X^N = -1
    for l, p in enumerate(c.primes):
        assert sq[l, 0] == p - 1 and (sq[l, 1:] == 0).all()


@pytest.mark.slow
@pytest.mark.parametrize("log_n", [16, 17])
def test_ntt_full_size_sampled(orc, log_n):
    # full sizes: sampled outputs against the definition, and the round trip
    primes = S.ntt_primes(log_n, 2, 60)
    c = orc.Ctx(log_n, primes[1:], primes[:1], 1)
    g = S.rng(300 + log_n)
    a = S.uniform_limbs(g, c.primes, c.n)
    A = c.ntt(a, [0, 1])
    js = sorted(set(int(v) for v in g.integers(0, c.n, 24)) | {0, 1, c.n - 1})
    for pidx in range(2):
        assert (c.ntt_def(a[pidx], pidx, js) == A[pidx, js]).all()
    assert (c.intt(A, [0, 1]) == a).all()


def test_automorph_eval_vs_coeff(orc):
    # EVAL permutation == NTT o (signed COEFF automorphism) o INTT  (reading 15)
    c = small_ctx(orc, 8, count=2, bits=50)
    g = S.rng(12)
    idx = [0, 1, 2]
    a = S.uniform_limbs(g, c.primes, c.n)
    A = c.ntt(a, idx)
    for k in (5, 25, 2 * c.n - 1, S.galois_rot(7, 8)):
        lhs = c.automorph(A, k)
        rhs = c.ntt(c.automorph_coeff(a, idx, k), idx)
        assert (lhs == rhs).all(), k
    assert (c.automorph(A, 1) == A).all()
    # group inverse: pi_k o pi_{k^-1} = id
    k = 5
    kinv = pow(k, -1, 2 * c.n)
    assert (c.automorph(c.automorph(A, k), kinv) == A).all()
    # COEFF form against the definition a(X^k) on a monomial: X^3 -> X^(3k mod 2N) with sign
    x = np.zeros((1, c.n), np.uint64)
    x[0, 3] = 1
    y = c.automorph_coeff(x, [0], 5)
    e = 15 % (2 * c.n)
    assert y[0, e] == 1
    x[0, 3] = 0
    x[0, 100] = 1
    y = c.automorph_coeff(x, [0], 5)
    assert y[0, 500 - 256] == c.primes[0] - 1   # 500 >= N=256 -> -X^(500-256)
