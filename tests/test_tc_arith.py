"""The integer identities the tensor-core kernels rely on (DESIGN.md §5 "Base conversion on the tensor
cores"), checked with Python integers on the host (-m "not gpu"): they are arithmetic facts independent
of the CUDA code, which the GPU parity tests then check end to end.

1. Byte-split contraction: for y = sum_a y_a 2^(8a) (bytes) and m_a = 2^(8a) M mod t,
   X' = sum_c 2^(8c) S_c with S_c = sum_{i,a} y_{i,a} byte_c(m_{i,a}) satisfies X' == sum_i y_i M_i (mod t),
   each S_c < 2^23 for up to 16 sources (s32 accumulators never overflow) and X' < 2^80.
2. The 14-instruction reduction: with mu = floor(2^80 / p), q = floor((X' >> 48) mu / 2^32) lies in
   [floor(X'/p) - 2, floor(X'/p)] for 2^49 < p < 2^60 and X' < 2^80, so X' - q p is in [0, 3p) and is
   exact in 64-bit arithmetic.
"""
import random

import pytest


def bytes_of(v, n=8):
    return [(v >> (8 * a)) & 0xFF for a in range(n)]


def bytesum(ys, ms, t):
    """X' of the byte-split contraction for sources ys (any 64-bit words) and matrix column ms (< t)."""
    S = [0] * 8
    for y, M in zip(ys, ms):
        yb = bytes_of(y)
        for a in range(8):
            ma = (M << (8 * a)) % t
            mb = bytes_of(ma)
            for c in range(8):
                S[c] += yb[a] * mb[c]
    return S, sum(s << (8 * c) for c, s in enumerate(S))


@pytest.mark.parametrize("nsrc", [1, 3, 9, 10, 16])
def test_byte_split_identity_and_bounds(nsrc):
    rng = random.Random(2507 + nsrc)
    for _ in range(200):
        t = rng.randrange(2**59, 2**60) | 1
        ys = [rng.randrange(2**64) for _ in range(nsrc)]          # any 64-bit word (lazy residues too)
        ms = [rng.randrange(t) for _ in range(nsrc)]
        S, X = bytesum(ys, ms, t)
        assert X % t == sum(y * M for y, M in zip(ys, ms)) % t
        assert max(S) < 2**23 and X < 2**80
    # worst case: every byte 0xFF
    t = 2**60 - 2**17 + 1
    S, X = bytesum([2**64 - 1] * 16, [t - 1] * 16, t)
    assert max(S) <= 16 * 8 * 255 * 255 < 2**23 and X < 2**80


def reduce14(X, p):
    """The integer steps of bytesum_reduce_c (modarith.cuh) on X' < 2^80."""
    mu = (1 << 80) // p
    top = X >> 48
    q = (top * mu) >> 32
    r = (X - q * p) % 2**64                                      # the kernel works modulo 2^64
    return q, r


@pytest.mark.parametrize("bits", [50, 55, 59, 60])
def test_bytesum_reduction_quotient_bound(bits):
    rng = random.Random(bits)
    edge = [0, 1, 2**80 - 1, 2**64, 2**64 - 1, 2**48, 2**79]
    for i in range(3000):
        p = rng.randrange(max(2**49 + 1, 2**(bits - 1)), 2**bits) | 1
        X = edge[i % len(edge)] if i < 4 * len(edge) else rng.randrange(2**80)
        q, r = reduce14(X, p)
        assert X // p - 2 <= q <= X // p
        assert r == X - q * p and 0 <= r < 3 * p and r % p == X % p


def test_twist_factorisation_small_ntt():
    """The tensor-core column pass factors the 256-row column transform into two 16-point rounds with a
    diagonal twist (W_B[b] = W_B[0] diag(d_b) forward); checked on a small prime with the same
    merged-twiddle Cooley-Tukey stages as the kernels."""
    p, logN, R = 786433, 16, 256
    N = 1 << logN
    g = 2
    while True:
        psi = pow(g, (p - 1) // (2 * N), p)
        if pow(psi, N, p) == p - 1:
            break
        g += 1
    brv = lambda x: int(format(x, "016b")[::-1], 2)
    psib = [pow(psi, brv(k), p) for k in range(R)]

    def stages(v, s0, s1):
        v = list(v)
        for s in range(s0, s1):
            m, t = 1 << s, R >> (s + 1)
            for i in range(m):
                w = psib[m + i]
                for j in range(2 * i * t, 2 * i * t + t):
                    X, Y = v[j], v[j + t] * w % p
                    v[j], v[j + t] = (X + Y) % p, (X - Y) % p
        return v

    def mat(s0, s1, base, stride):
        M = [[0] * 16 for _ in range(16)]
        for k in range(16):
            e = [0] * R
            e[base + stride * k] = 1
            out = stages(e, s0, s1)
            for kk in range(16):
                M[kk][k] = out[base + stride * kk]
        return M

    WA, WB0 = mat(0, 4, 0, 16), mat(4, 8, 0, 1)
    assert all(mat(0, 4, r0, 16) == WA for r0 in (1, 7, 15))
    rng = random.Random(1)
    x = [rng.randrange(p) for _ in range(R)]
    ref = stages(x, 0, 8)
    y = [0] * R
    for r0 in range(16):
        for kk in range(16):
            y[r0 + 16 * kk] = sum(WA[kk][k] * x[r0 + 16 * k] for k in range(16)) % p
    z = [0] * R
    for b in range(16):
        Wb = mat(4, 8, 16 * b, 1)
        d = [Wb[0][k] * pow(WB0[0][k], p - 2, p) % p for k in range(16)]
        for kk in range(16):
            z[16 * b + kk] = sum(WB0[kk][k] * d[k] * y[16 * b + k] for k in range(16)) % p
    assert z == ref
