// modarith.cuh -- 64-bit modular arithmetic for sm_100a (§3.6.2, tab:mod_red).
//
// Residues are u64 modulo primes p < 2^60.  Internal ranges are lazy ([0,2p) / [0,4p)), canonical
// [0,p) at every API boundary and for every base-conversion input (SURVEY.md §8(c) readings 4, 16).
//
//  * Shoup multiplication (tab:mod_red "1 wide + 2 low"): w' = floor(w * 2^64 / p), any x < 2^64:
//      q = hi64(x * w'),  r = lo64(x * w) - lo64(q * p)  in [0, 2p).
//  * 128-bit reduction of base-conversion / inner-product sums: the products are formed from
//    30-bit halves (y = yh*2^30 + yl) so that every partial product is one IMAD.WIDE.U32 with a
//    64-bit accumulator (carry-free for up to 16 terms), then the 128-bit sum is reduced with two
//    Shoup steps:  X = hi*2^64 + lo,  X mod p = shoup(hi, 2^64 mod p) + shoup(lo, 1)  in [0, 4p).
#pragma once
#include <stdint.h>

typedef uint64_t u64;
typedef uint32_t u32;

#define HKS_DEV __device__ __forceinline__

HKS_DEV u64 mulhi64(u64 a, u64 b) { return __umul64hi(a, b); }

// x * w mod p in [0, 2p), w' = floor(w 2^64 / p).
HKS_DEV u64 shoup_lazy(u64 x, u64 w, u64 wp, u64 p) {
    u64 q = mulhi64(x, wp);
    return x * w - q * p;
}

HKS_DEV u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }

HKS_DEV u64 shoup(u64 x, u64 w, u64 wp, u64 p) { return csub(shoup_lazy(x, w, wp, p), p); }

// Per-prime constants used by the reductions.
struct PrimeConst {
    u64 p;       // modulus
    u64 r64;     // 2^64 mod p
    u64 r64p;    // Shoup companion of r64
    u64 one_p;   // floor(2^64 / p): Shoup companion of 1
    u64 mu80;    // floor(2^80 / p) (< 2^32 for p > 2^48): byte-sum reduction of the tensor-pipe BConv
};

// 128-bit accumulator of 30-bit-split products:  X = s2*2^60 + (s1a + s1b)*2^30 + s0.
struct Acc30 {
    u64 s0, s1a, s1b, s2;
};

HKS_DEV void acc_zero(Acc30 &a) { a.s0 = a.s1a = a.s1b = a.s2 = 0; }

// a += y * m with y = (yh, yl), m = (mh, ml) 30-bit halves.  4 IMAD.WIDE.U32 (PTX, so that the
// compiler neither re-materialises the split nor routes the accumulators through extra adds).
HKS_DEV void mad_wide(u64 &acc, u32 a, u32 b) { asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b)); }
HKS_DEV u64 mul_wide(u32 a, u32 b) {
    u64 r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}

HKS_DEV void acc_mac(Acc30 &a, u32 yl, u32 yh, u32 ml, u32 mh) {
    mad_wide(a.s0, yl, ml);
    mad_wide(a.s1a, yl, mh);
    mad_wide(a.s1b, yh, ml);
    mad_wide(a.s2, yh, mh);
}

// first term of a chain: a = y * m
HKS_DEV void acc_first(Acc30 &a, u32 yl, u32 yh, u32 ml, u32 mh) {
    a.s0 = mul_wide(yl, ml);
    a.s1a = mul_wide(yl, mh);
    a.s1b = mul_wide(yh, ml);
    a.s2 = mul_wide(yh, mh);
}

HKS_DEV void split30(u64 y, u32 &lo, u32 &hi) {
    u32 l, h;
    asm("{\n\t.reg .u32 a, b;\n\tmov.b64 {a, b}, %2;\n\tand.b32 %0, a, 0x3fffffff;\n\tshf.r.clamp.b32 %1, a, b, 30;\n\t}"
        : "=r"(l), "=r"(h) : "l"(y));
    lo = l;
    hi = h;
}

// 128-bit value of an Acc30 accumulator:  s0 + (s1a + s1b) 2^30 + s2 2^60.
HKS_DEV void acc_to128(const Acc30 &a, u64 &lo, u64 &hi) {
    u64 t;
    lo = a.s0;
    hi = 0;
    t = a.s1a << 30; lo += t; hi += (lo < t); hi += a.s1a >> 34;
    t = a.s1b << 30; lo += t; hi += (lo < t); hi += a.s1b >> 34;
    t = a.s2 << 60;  lo += t; hi += (lo < t); hi += a.s2 >> 4;
}

// ---- Karatsuba accumulation (3 IMAD.WIDE per MAC): y m = yl ml + ((yl+yh)(ml+mh) - yl ml - yh mh) 2^30
// + yh mh 2^60.  (yl+yh), (ml+mh) < 2^31, so a middle product is < 2^62 and each of the three middle
// accumulators (terms i = 0, 1, 2 mod 3) stays below 2^64 for up to 12 terms; s0, s2 < 16 * 2^60.
struct AccK {
    u64 s0, s2, m0, m1, m2;
};

template <int I>
HKS_DEV void acck_mac(AccK &a, u32 yl, u32 yh, u32 ys, u32 ml, u32 mh, u32 ms) {
    if (I == 0) {
        a.s0 = mul_wide(yl, ml);
        a.s2 = mul_wide(yh, mh);
    } else {
        mad_wide(a.s0, yl, ml);
        mad_wide(a.s2, yh, mh);
    }
    if (I % 3 == 0) {
        if (I == 0) a.m0 = mul_wide(ys, ms); else mad_wide(a.m0, ys, ms);
    } else if (I % 3 == 1) {
        if (I == 1) a.m1 = mul_wide(ys, ms); else mad_wide(a.m1, ys, ms);
    } else {
        if (I == 2) a.m2 = mul_wide(ys, ms); else mad_wide(a.m2, ys, ms);
    }
}

// 128-bit value s0 + (m0 + m1 + m2 - s0 - s2) 2^30 + s2 2^60 for a chain of n terms
HKS_DEV void acck_to128(const AccK &a, int n, u64 &lo, u64 &hi) {
    // mid = m0 + m1 + m2 - s0 - s2  (< 2^66 as a 128-bit intermediate; the true value is < 2^65)
    u64 mlo = a.m0, mhi = 0, t;
    if (n > 1) { t = a.m1; mlo += t; mhi += (mlo < t); }
    if (n > 2) { t = a.m2; mlo += t; mhi += (mlo < t); }
    mhi -= (mlo < a.s0); mlo -= a.s0;
    mhi -= (mlo < a.s2); mlo -= a.s2;
    lo = a.s0;
    hi = 0;
    t = mlo << 30; lo += t; hi += (lo < t); hi += (mlo >> 34) | (mhi << 30);
    t = a.s2 << 60; lo += t; hi += (lo < t); hi += a.s2 >> 4;
}

// ---- FP64-pipe partial dot products (k_bconv_fp): 60-bit operands as three exact 20-bit limbs in
// doubles; every product < 2^40 and every partial sum < 2^46 is an integer below 2^53, so DFMA is
// exact.  Five accumulators C_c = sum_{a+b=c} Y_a M_b give X = sum_c C_c 2^(20c).
struct AccF {
    double c[5];
};

HKS_DEV double exact_dbl(u32 v) {   // v < 2^52: 2^52 + v has v as its mantissa
    return __longlong_as_double(0x4330000000000000ll | (long long)v) - 4503599627370496.0;
}

HKS_DEV void split20d(u64 y, double &y0, double &y1, double &y2) {
    y0 = exact_dbl((u32)y & 0xfffffu);
    y1 = exact_dbl((u32)(y >> 20) & 0xfffffu);
    y2 = exact_dbl((u32)(y >> 40));
}

HKS_DEV void accf_first(AccF &A, double y0, double y1, double y2, double m0, double m1, double m2) {
    A.c[0] = y0 * m0;
    A.c[1] = fma(y1, m0, y0 * m1);
    A.c[2] = fma(y2, m0, fma(y1, m1, y0 * m2));
    A.c[3] = fma(y2, m1, y1 * m2);
    A.c[4] = y2 * m2;
}

HKS_DEV void accf_mac(AccF &A, double y0, double y1, double y2, double m0, double m1, double m2) {
    A.c[0] = fma(y0, m0, A.c[0]);
    A.c[1] = fma(y1, m0, fma(y0, m1, A.c[1]));
    A.c[2] = fma(y2, m0, fma(y1, m1, fma(y0, m2, A.c[2])));
    A.c[3] = fma(y2, m1, fma(y1, m2, A.c[3]));
    A.c[4] = fma(y2, m2, A.c[4]);
}

HKS_DEV u64 dbl_int(double c) {    // c integral in [0, 2^52)
    return (u64)(__double_as_longlong(c + 4503599627370496.0) - 0x4330000000000000ll);
}

// (lo, hi) += sum_c C_c 2^(20c)
HKS_DEV void accf_add128(const AccF &A, u64 &lo, u64 &hi) {
    const u64 c0 = dbl_int(A.c[0]), c1 = dbl_int(A.c[1]), c2 = dbl_int(A.c[2]), c3 = dbl_int(A.c[3]),
              c4 = dbl_int(A.c[4]);
    u64 t;
    t = c0;       lo += t; hi += (lo < t);
    t = c1 << 20; lo += t; hi += (lo < t); hi += c1 >> 44;
    t = c2 << 40; lo += t; hi += (lo < t); hi += c2 >> 24;
    t = c3 << 60; lo += t; hi += (lo < t); hi += c3 >> 4;
    hi += c4 << 16;
}

// canonical X mod p for the accumulated 128-bit value (< 2^124, i.e. <= 16 terms of 60x60 bits).
// (Defined after shoup_approx below.)
HKS_DEV u64 acc_reduce(const Acc30 &a, const PrimeConst &c);

// X = hi 2^64 + lo (hi < 2^62) reduced to [0, 8p) with two approximate-quotient Shoup steps.
// (Defined after shoup_approx below.)
HKS_DEV u64 acc_reduce_lazy(const Acc30 &a, const PrimeConst &c);

// Per-prime constants of the lazy butterflies.
struct NttMod {
    u64 p, np;       // p and 2^64 - p
    u64 two_p, four_p, eight_p;
    u32 h4;          // (4p) >> 32: hi-word threshold of the one-instruction range test
    u64 zh;          // 0, but opaque to ptxas (derived from p): see lazy_add
};

HKS_DEV NttMod make_nttmod(u64 p) {
    NttMod m;
    m.p = p;
    m.np = 0 - p;
    m.two_p = 2 * p;
    m.four_p = 4 * p;
    m.eight_p = 8 * p;
    m.h4 = (u32)((4 * p) >> 32);
    m.zh = (u64)(u32)(p >> 63) << 32;   // p < 2^60: zero
    return m;
}

// x + y for the butterflies.  ptxas lowers a two-operand 64-bit add to IADD3 + IMAD.X, and IMAD.X issues
// on the FMA-heavy pipe of the Shoup products (~1.25 per butterfly).  With OPQ the opaque zero m.zh joins
// the high word, so the carry-add is a three-input IADD3.X on the ALU pipe, at no extra instruction.
// Measured per pass: faster for the inverse row pass only (ptxas then re-balances the other
// passes with IMAD.MOV and select instructions), so the choice is a template parameter of the butterflies.
template <bool OPQ>
HKS_DEV u64 lazy_add(u64 x, u64 y, const NttMod &m) { return OPQ ? x + y + m.zh : x + y; }

// Shoup product with an approximate quotient: three 32x32 partial products of y * w' (the
// low x low one dropped), so q is short by 0..2 and the result is y*w mod p in [0, 4p) for any
// y < 2^64.  r = y*w - q*p is formed as y*w + q*(2^64 - p) mod 2^64.
HKS_DEV u64 shoup_approx(u64 y, u64 w, u64 wp, u64 np) {
#ifdef HKS_EXACT_SHOUP
    return y * w + __umul64hi(y, wp) * np;      // [0, 2p)
#elif !defined(HKS_C_SHOUP)
    // 2 IMAD.HI + 3 IMAD.WIDE + 4 IMAD (28 FMA-pipe cycles per warp on sm_100); the 33-bit sum of
    // the two high halves is a plain 64-bit add so that it lands on the ALU pipe.
    u64 r;
    asm("{\n\t"
        ".reg .u32 yl, yh, wl, wh, pl, ph, nl, nh, t1, t3, ql, qh, rl, rh;\n\t"
        ".reg .u64 a, b, mid, q, rr;\n\t"
        "mov.b64 {yl, yh}, %1;\n\t"
        "mov.b64 {wl, wh}, %2;\n\t"
        "mov.b64 {pl, ph}, %3;\n\t"
        "mov.b64 {nl, nh}, %4;\n\t"
        "mul.hi.u32 t1, yh, pl;\n\t"
        "mul.hi.u32 t3, yl, ph;\n\t"
        "cvt.u64.u32 a, t1;\n\t"
        "cvt.u64.u32 b, t3;\n\t"
        "add.u64 mid, a, b;\n\t"
        "mad.wide.u32 q, yh, ph, mid;\n\t"
        "mov.b64 {ql, qh}, q;\n\t"
        "mul.wide.u32 rr, yl, wl;\n\t"
        "mad.wide.u32 rr, ql, nl, rr;\n\t"
        "mov.b64 {rl, rh}, rr;\n\t"
        "mad.lo.u32 rh, yh, wl, rh;\n\t"
        "mad.lo.u32 rh, yl, wh, rh;\n\t"
        "mad.lo.u32 rh, qh, nl, rh;\n\t"
        "mad.lo.u32 rh, ql, nh, rh;\n\t"
        "mov.b64 %0, {rl, rh};\n\t"
        "}"
        : "=l"(r) : "l"(y), "l"(w), "l"(wp), "l"(np));
    return r;
#else
    const u32 yl = (u32)y, yh = (u32)(y >> 32), wl = (u32)wp, wh = (u32)(wp >> 32);
    const u64 mid = (u64)__umulhi(yh, wl) + __umulhi(yl, wh);
    const u64 q = (u64)yh * wh + mid;
    return y * w + q * np;
#endif
}

// x >= 4p (tested on the high word only) ? x - 4p : x.  For x < 8p + 2^32 the result is < 4p + 2^32.
template <bool OPQ = false>
HKS_DEV u64 lazy_sub4p(u64 x, const NttMod &m) {
    u64 r = x;
    if (!OPQ) {
    asm("{\n\t"
        ".reg .pred p;\n\t"
        ".reg .u32 xl, xh, fl, fh;\n\t"
        "mov.b64 {xl, xh}, %0;\n\t"
        "mov.b64 {fl, fh}, %2;\n\t"
        "setp.gt.u32 p, xh, %1;\n\t"
        "@p sub.cc.u32 xl, xl, fl;\n\t"
        "@p subc.u32 xh, xh, fh;\n\t"
        "mov.b64 %0, {xl, xh};\n\t"
        "}"
        : "+l"(r) : "r"(m.h4), "l"(m.four_p));
    return r;
    }
    // OPQ: x - 4p with the opaque zero in its high word (see lazy_add): a three-input IADD3.X, not IMAD.X
    asm("{\n\t"
        ".reg .pred p;\n\t"
        ".reg .u32 xl, xh, fl, fh, zl, zh, dl, dh;\n\t"
        "mov.b64 {xl, xh}, %0;\n\t"
        "mov.b64 {fl, fh}, %2;\n\t"
        "mov.b64 {zl, zh}, %3;\n\t"
        "setp.gt.u32 p, xh, %1;\n\t"
        "sub.cc.u32 dl, xl, fl;\n\t"
        "subc.u32 dh, xh, fh;\n\t"
        "add.u32 dh, dh, zh;\n\t"
        "selp.b32 xl, dl, xl, p;\n\t"
        "selp.b32 xh, dh, xh, p;\n\t"
        "mov.b64 %0, {xl, xh};\n\t"
        "}"
        : "+l"(r) : "r"(m.h4), "l"(m.four_p), "l"(m.zh));
    return r;
}

// Forward CT butterfly on the lazy range [0, 8p + 2^32):  X' = x + t, Y' = x - t + 4p with
// x = X reduced below 4p + 2^32 and t = Y*w in [0, 4p).  Both outputs stay in [0, 8p + 2^32).
template <bool OPQ = false>
HKS_DEV void ct_lazy(u64 &X, u64 &Y, u64 w, u64 wp, const NttMod &m) {
    const u64 x = lazy_sub4p<OPQ>(X, m);
    const u64 t = shoup_approx(Y, w, wp, m.np);
    X = lazy_add<OPQ>(x, t, m);
    Y = x - t + m.four_p;
}

// Inverse GS butterfly.  Inputs < 4p + c with c <= 2^(32+s) after s stages (c < 4p for every
// supported N): X' = X + Y reduced by 4p on the high-word test (< 4p + 2c), Y' = (X - Y + 8p)*w in
// [0, 4p).
template <bool OPQ = false>
HKS_DEV void gs_lazy(u64 &X, u64 &Y, u64 w, u64 wp, const NttMod &m) {
    const u64 x = X, y = Y;
    X = lazy_sub4p<OPQ>(lazy_add<OPQ>(x, y, m), m);
    Y = shoup_approx(x - y + m.eight_p, w, wp, m.np);
}

// canonical residue of x < 8p + 2^33
HKS_DEV u64 canon8(u64 x, const NttMod &m) {
    x = csub(x, m.four_p);
    x = csub(x, m.two_p);
    x = csub(x, m.p);
    return csub(x, m.p);
}

// Forward Cooley-Tukey butterfly, Harvey lazy form: X, Y in [0, 4p) -> [0, 4p).
HKS_DEV void ct_bfly(u64 &X, u64 &Y, u64 w, u64 wp, u64 p, u64 two_p) {
    u64 x = csub(X, two_p);
    u64 t = shoup_lazy(Y, w, wp, p);
    X = x + t;
    Y = x - t + two_p;
}

// Inverse Gentleman-Sande butterfly: X, Y in [0, 2p) -> [0, 2p).
HKS_DEV void gs_bfly(u64 &X, u64 &Y, u64 w, u64 wp, u64 p, u64 two_p) {
    u64 x = X, y = Y;
    X = csub(x + y, two_p);
    Y = shoup_lazy(x - y + two_p, w, wp, p);
}

// bit reversal of the low `bits` bits
HKS_DEV u32 brev_bits(u32 x, u32 bits) { return __brev(x) >> (32 - bits); }

// EVAL-form automorphism source index (SURVEY.md §8(c) reading 15):
//   j' with 2 brv(j') + 1 = k (2 brv(j) + 1) mod 2N.
HKS_DEV u32 automorph_src(u32 j, u32 log_n, u64 galois) {
    u32 two_n_mask = (2u << log_n) - 1;
    u32 e = ((u32)galois * (2u * brev_bits(j, log_n) + 1u)) & two_n_mask;
    return brev_bits((e - 1u) >> 1, log_n);
}


// lo mod p in [0, 4p) for p > 2^32: one_p = floor(2^64/p) < 2^32, so the quotient estimate is one
// 32x32 high product of lo's high word (short by at most 3), and lo - q p needs one IMAD.WIDE + IMAD.
HKS_DEV u64 mod64_lazy(u64 lo, const PrimeConst &c) {
    if (c.one_p >> 32) return shoup_approx(lo, 1, c.one_p, 0 - c.p);   // p < 2^32: generic path
    const u32 q = __umulhi((u32)(lo >> 32), (u32)c.one_p);
    return lo + (u64)q * (0 - c.p);
}

// X = hi 2^64 + lo (hi < 2^62) reduced to [0, 8p): hi (2^64 mod p) by an approximate Shoup step,
// lo by mod64_lazy.
HKS_DEV u64 reduce128_lazy(u64 lo, u64 hi, const PrimeConst &c) {
    return shoup_approx(hi, c.r64, c.r64p, 0 - c.p) + mod64_lazy(lo, c);
}

HKS_DEV u64 reduce128(u64 lo, u64 hi, const PrimeConst &c) {
    u64 r = reduce128_lazy(lo, hi, c);   // [0, 8p)
    r = csub(r, 4 * c.p);
    r = csub(r, 2 * c.p);
    return csub(r, c.p);
}

// x * y mod p, canonical, for x, y < 2^60 (one 128-bit product, one reduction)
HKS_DEV u64 mulmod_full(u64 x, u64 y, const PrimeConst &c) { return reduce128(x * y, __umul64hi(x, y), c); }

// (x0 y0 + x1 y1) mod p, canonical, for operands < 2^60 (128-bit sum < 2^121, one reduction)
HKS_DEV u64 mul2mod_full(u64 x0, u64 y0, u64 x1, u64 y1, const PrimeConst &c) {
    const u64 l0 = x0 * y0, l1 = x1 * y1, lo = l0 + l1;
    const u64 hi = __umul64hi(x0, y0) + __umul64hi(x1, y1) + (lo < l0 ? 1 : 0);
    return reduce128(lo, hi, c);
}

// SwitchModulo of t in [0, qs) from modulus qs into p, centered representative (t if 2t < qs, else
// t - qs): the Rescale prologue (reading 15).  qs_mod_p = qs mod p.
HKS_DEV u64 switch_centered(u64 t, u64 qs, u64 qs_mod_p, const PrimeConst &c) {
    u64 r = csub(csub(mod64_lazy(t, c), 2 * c.p), c.p);
    if (t > (qs >> 1)) r = r >= qs_mod_p ? r - qs_mod_p : r + c.p - qs_mod_p;
    return r;
}

// ---- base conversion on the tensor pipe (k_bconv_mma): byte-split products -------------------
// Legacy warp-level integer MMA (SASS IMMA): D(16x8, s32) += A(16xK, u8, row) * B(Kx8, u8, col).
HKS_DEV void mma_u8_k32(int (&d)[4], const u32 (&a)[4], u32 b0, u32 b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
HKS_DEV void mma_u8_k16(int (&d)[4], u32 a0, u32 a1, u32 b0) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(b0));
}

// y * w mod p in [0, 2p) for a 32-bit multiplier y (exact Shoup quotient from two 32-bit products).
HKS_DEV u64 shoup_u32(u32 y, u64 w, u64 wp, u64 np) {
    const u32 t1 = __umulhi(y, (u32)wp);
    const u32 q = (u32)(((u64)y * (u32)(wp >> 32) + t1) >> 32);
    const u64 r = (u64)y * (u32)w + (u64)q * (u32)np;
    const u32 rh = (u32)(r >> 32) + y * (u32)(w >> 32) + q * (u32)(np >> 32);
    return ((u64)rh << 32) | (u32)r;
}

// X' = sum_c S_c 2^(8c) (S_c < 2^23, c = 0..7, so X' < 2^80) reduced modulo p, 2^49 < p < 2^60:
// [0, 3p) lazily, else canonical.  X' = a + T67 2^48 with a = T01 + T23 2^16 + T45 2^32 < 2^64 and
// T_{c,c+1} = S_c + S_{c+1} 2^8 < 2^32.  Quotient estimate q = floor((X' >> 48) mu / 2^32) with
// mu = floor(2^80 / p): q <= X'/p < q + 3 (truncations cost < 1 + 2^48/p), so X' - q p < 3p is
// exact in 64-bit arithmetic.  The byte combinations are funnel shifts and adds, which ptxas emits as
// LEA.HI on the ALU pipe (a plain shl + add, or a mad by 256, becomes an IMAD on the FMA-heavy pipe),
// so that the heavy pipe carries little more than the quotient step: ~12 SASS instructions per output.
template <bool LAZY>
HKS_DEV u64 bytesum_reduce_c(u32 s0, u32 s1, u32 s2, u32 s3, u32 s4, u32 s5, u32 s6, u32 s7, u64 np, u32 mu) {
    u64 r;
    asm("{\n\t"
        ".reg .u32 t01, t23, t45, t67, x, y, al, ah, top, q, n0, n1, rl, rh;\n\t"
        ".reg .u64 aa, rr;\n\t"
        "shf.l.wrap.b32 x, %2, %2, 8;\n\t"
        "add.u32 t01, x, %1;\n\t"
        "shf.l.wrap.b32 x, %4, %4, 8;\n\t"
        "add.u32 t23, x, %3;\n\t"
        "shf.l.wrap.b32 x, %6, %6, 8;\n\t"
        "add.u32 t45, x, %5;\n\t"
        "shf.l.wrap.b32 x, %8, %8, 8;\n\t"
        "add.u32 t67, x, %7;\n\t"
        "shl.b32 x, t23, 16;\n\t"
        "shr.u32 y, t23, 16;\n\t"
        "add.cc.u32 al, t01, x;\n\t"
        "addc.u32 ah, t45, y;\n\t"                 // a = (al, ah)
        "shr.u32 x, ah, 16;\n\t"
        "add.u32 top, x, t67;\n\t"                 // X' >> 48
        "shf.l.clamp.b32 x, 0, t67, 16;\n\t"
        "add.u32 ah, ah, x;\n\t"                   // X' mod 2^64
        "mul.hi.u32 q, top, %10;\n\t"
        "mov.b64 {n0, n1}, %9;\n\t"                // 2^64 - p
        "mov.b64 aa, {al, ah};\n\t"
        "mad.wide.u32 rr, q, n0, aa;\n\t"
        "mov.b64 {rl, rh}, rr;\n\t"
        "mad.lo.u32 rh, q, n1, rh;\n\t"
        "mov.b64 %0, {rl, rh};\n\t"
        "}"
        : "=l"(r)
        : "r"(s0), "r"(s1), "r"(s2), "r"(s3), "r"(s4), "r"(s5), "r"(s6), "r"(s7), "l"(np), "r"(mu));
    if (!LAZY) {
        const u64 p = 0 - np;
        r = csub(r, 2 * p);
        r = csub(r, p);
    }
    return r;
}
template <bool LAZY>
HKS_DEV u64 bytesum_reduce(u32 s0, u32 s1, u32 s2, u32 s3, u32 s4, u32 s5, u32 s6, u32 s7, const PrimeConst &c) {
    return bytesum_reduce_c<LAZY>(s0, s1, s2, s3, s4, s5, s6, s7, 0 - c.p, (u32)c.mu80);
}
template <bool LAZY>
HKS_DEV u64 bytesum_reduce_c(const u32 (&v)[8], u64 np, u32 mu) {
    return bytesum_reduce_c<LAZY>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], np, mu);
}

HKS_DEV u64 acc_reduce_lazy(const Acc30 &a, const PrimeConst &c) {
    u64 lo, hi;
    acc_to128(a, lo, hi);
    return reduce128_lazy(lo, hi, c);
}

HKS_DEV u64 acc_reduce(const Acc30 &a, const PrimeConst &c) {
    u64 lo, hi;
    acc_to128(a, lo, hi);
    return reduce128(lo, hi, c);
}
