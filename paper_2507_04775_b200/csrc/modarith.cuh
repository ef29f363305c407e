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
};

// 128-bit accumulator of 30-bit-split products:  X = s2*2^60 + (s1a + s1b)*2^30 + s0.
struct Acc30 {
    u64 s0, s1a, s1b, s2;
};

HKS_DEV void acc_zero(Acc30 &a) { a.s0 = a.s1a = a.s1b = a.s2 = 0; }

// a += y * m with y = (yh, yl), m = (mh, ml) 30-bit halves.  4 IMAD.WIDE.U32.
HKS_DEV void acc_mac(Acc30 &a, u32 yl, u32 yh, u32 ml, u32 mh) {
    a.s0 += (u64)yl * ml;
    a.s1a += (u64)yl * mh;
    a.s1b += (u64)yh * ml;
    a.s2 += (u64)yh * mh;
}

HKS_DEV void split30(u64 y, u32 &lo, u32 &hi) {
    lo = (u32)y & 0x3fffffffu;
    hi = (u32)(y >> 30);
}

// canonical X mod p for the accumulated 128-bit value (< 2^124, i.e. <= 16 terms of 60x60 bits).
HKS_DEV u64 acc_reduce(const Acc30 &a, const PrimeConst &c) {
    // lo/hi of s0 + (s1a << 30) + (s1b << 30) + (s2 << 60)
    u64 lo = a.s0, hi = 0, t;
    t = a.s1a << 30; lo += t; hi += (lo < t); hi += a.s1a >> 34;
    t = a.s1b << 30; lo += t; hi += (lo < t); hi += a.s1b >> 34;
    t = a.s2 << 60;  lo += t; hi += (lo < t); hi += a.s2 >> 4;
    u64 r = shoup_lazy(hi, c.r64, c.r64p, c.p) + (lo - mulhi64(lo, c.one_p) * c.p);   // [0, 4p)
    r = csub(r, 2 * c.p);
    return csub(r, c.p);
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
