/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for hybrid key switching.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2507_04775_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant generator with it.
 *
 * Every modular operation is `%` on unsigned __int128 -- no Barrett, no Shoup, no
 * lazy ranges, no blocking or fusion.  Each function cites the passage it follows:
 *   PAPER.md  = /root/reference/PAPER.md (FIDESlib, arXiv 2507.04775), line + section
 *   SPEC.md   = /root/reference/SPEC.md, line + module
 *   SURVEY.md = /root/repo/SURVEY.md §8(c), the readings adopted where the paper is silent.
 *
 * Conventions (SURVEY.md §8(c) readings 1, 2, 3, 11, 15):
 *   psi_m   = the minimal primitive 2N-th root of unity mod prime m.
 *   EVAL    = bit-reversed evaluation order: ahat[j] = a(psi^(2*brv(j)+1)).
 *   COEFF   = natural coefficient order; INTT includes N^-1.
 *   Extended limb order: Q_0..Q_l, P_0..P_{K-1}; key limb index of P_k is L+1+k.
 *   Digit j = chain limbs [j*alpha, min((j+1)*alpha, l+1)), alpha = ceil((L+1)/dnum).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;
typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- scalars */

static u64 mulmod(u64 a, u64 b, u64 p) { return (u64)(((u128)a * b) % p); }
static u64 addmod(u64 a, u64 b, u64 p) { return (u64)(((u128)a + b) % p); }
static u64 submod(u64 a, u64 b, u64 p) { return (u64)(((u128)a + p - (b % p)) % p); }

static u64 powmod(u64 a, u64 e, u64 p) {
    u64 r = 1 % p;
    a %= p;
    while (e) {
        if (e & 1) r = mulmod(r, a, p);
        a = mulmod(a, a, p);
        e >>= 1;
    }
    return r;
}

/* Fermat inverse; p prime, a != 0 mod p. */
static u64 invmod(u64 a, u64 p) { return powmod(a, p - 2, p); }

/* deterministic Miller-Rabin for 64-bit n */
int or_is_prime(u64 n) {
    static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n % bases[i] == 0) return n == bases[i];
    }
    u64 d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int composite = 1;
        for (int r = 1; r < s; r++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { composite = 0; break; }
        }
        if (composite) return 0;
    }
    return 1;
}

/* SURVEY.md §8(c) reading 1 (Table 2 "2n-th root of unity"):
 * psi = the smallest x in [2,p) with x^N = -1 (mod p).  All such x are psi0^k for
 * odd k < 2N, psi0 any one of them, so we enumerate those N candidates. */
u64 or_min_psi(u64 p, u32 n) {
    u64 psi0 = 0;
    for (u64 x = 2; x < p; x++) {
        u64 c = powmod(x, (p - 1) / (2 * (u64)n), p);
        if (powmod(c, n, p) == p - 1) { psi0 = c; break; }
    }
    if (!psi0) return 0;
    u64 sq = mulmod(psi0, psi0, p), cur = psi0, best = psi0;
    for (u64 k = 1; k < 2 * (u64)n; k += 2) {
        if (cur < best) best = cur;
        cur = mulmod(cur, sq, p);
    }
    return best;
}

static u32 brv(u32 x, u32 bits) {
    u32 r = 0;
    for (u32 i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}

/* ---------------------------------------------------------------- context */

typedef struct or_ctx {
    u32 log_n, n, nq, np, dnum, alpha;
    u64 *m;       /* q_0..q_L, p_0..p_{K-1} */
    u64 *psi;     /* per prime */
} or_ctx;

void or_ctx_free(or_ctx *c) {
    if (!c) return;
    free(c->m);
    free(c->psi);
    free(c);
}

/* returns NULL on invalid parameters (not prime, not 1 mod 2N, >= 2^60, duplicate) */
or_ctx *or_ctx_new(u32 log_n, const u64 *q, u32 nq, const u64 *p, u32 np, u32 dnum) {
    if (log_n < 1 || log_n > 20 || nq < 1 || np < 1 || dnum < 1 || dnum > nq) return NULL;
    or_ctx *c = (or_ctx *)calloc(1, sizeof(or_ctx));
    c->log_n = log_n;
    c->n = 1u << log_n;
    c->nq = nq;
    c->np = np;
    c->dnum = dnum;
    c->alpha = (nq + dnum - 1) / dnum;
    c->m = (u64 *)malloc(sizeof(u64) * (nq + np));
    c->psi = (u64 *)malloc(sizeof(u64) * (nq + np));
    for (u32 i = 0; i < nq; i++) c->m[i] = q[i];
    for (u32 k = 0; k < np; k++) c->m[nq + k] = p[k];
    for (u32 i = 0; i < nq + np; i++) {
        u64 mi = c->m[i];
        int bad = mi >= (1ull << 60) || !or_is_prime(mi) || (mi - 1) % (2 * (u64)c->n) != 0;
        for (u32 j = 0; j < i; j++) bad |= c->m[j] == mi;
        if (bad) { or_ctx_free(c); return NULL; }
        c->psi[i] = or_min_psi(mi, c->n);
    }
    return c;
}

u64 or_ctx_psi(const or_ctx *c, u32 idx) { return c->psi[idx]; }
u32 or_ctx_alpha(const or_ctx *c) { return c->alpha; }

/* number of active digits at level l: beta = ceil((l+1)/alpha) */
static u32 beta_of(const or_ctx *c, u32 level) { return (level + 1 + c->alpha - 1) / c->alpha; }
u32 or_beta(const or_ctx *c, u32 level) { return beta_of(c, level); }

static void digit_range(const or_ctx *c, u32 level, u32 j, u32 *lo, u32 *hi) {
    *lo = j * c->alpha;
    u32 h = (j + 1) * c->alpha;
    *hi = h < level + 1 ? h : level + 1;
}

/* extended-limb position (0..l+K) -> prime index into c->m */
static u32 ext_prime(const or_ctx *c, u32 level, u32 t) { return t <= level ? t : c->nq + (t - level - 1); }

/* ---------------------------------------------------------------- NTT */

/* Forward negacyclic NTT of one limb, textbook form (§3.6.4):
 *   ahat[j] = sum_i a_i psi^(i(2brv(j)+1))
 * computed as b_i = a_i psi^i (twist), B = cyclic DFT of b with omega = psi^2 by the
 * iterative radix-2 FFT (bit-reverse copy, then butterflies), ahat[j] = B[brv(j)]. */
static void ntt_one(u64 *a, u32 log_n, u64 p, u64 psi) {
    u32 n = 1u << log_n;
    u64 *b = (u64 *)malloc(sizeof(u64) * n);
    u64 *B = (u64 *)malloc(sizeof(u64) * n);
    u64 pw = 1;
    for (u32 i = 0; i < n; i++) { b[i] = mulmod(a[i], pw, p); pw = mulmod(pw, psi, p); }
    for (u32 i = 0; i < n; i++) B[brv(i, log_n)] = b[i];
    u64 omega = mulmod(psi, psi, p);
    for (u32 s = 1; s <= log_n; s++) {
        u32 m = 1u << s;
        u64 wm = powmod(omega, n / m, p);
        for (u32 k = 0; k < n; k += m) {
            u64 w = 1;
            for (u32 j = 0; j < m / 2; j++) {
                u64 t = mulmod(w, B[k + j + m / 2], p);
                u64 u = B[k + j];
                B[k + j] = addmod(u, t, p);
                B[k + j + m / 2] = submod(u, t, p);
                w = mulmod(w, wm, p);
            }
        }
    }
    for (u32 j = 0; j < n; j++) a[j] = B[brv(j, log_n)];
    free(b);
    free(B);
}

/* Inverse (§3.6.4): a_i = N^-1 psi^-i sum_k B[k] omega^-ik,
 * with B[k] = ahat[brv(k)] -- the exact inverse of ntt_one, including N^-1. */
static void intt_one(u64 *a, u32 log_n, u64 p, u64 psi) {
    u32 n = 1u << log_n;
    u64 *B = (u64 *)malloc(sizeof(u64) * n);
    u64 *C = (u64 *)malloc(sizeof(u64) * n);
    for (u32 k = 0; k < n; k++) B[k] = a[brv(k, log_n)];
    for (u32 i = 0; i < n; i++) C[brv(i, log_n)] = B[i];
    u64 omega_inv = invmod(mulmod(psi, psi, p), p);
    for (u32 s = 1; s <= log_n; s++) {
        u32 m = 1u << s;
        u64 wm = powmod(omega_inv, n / m, p);
        for (u32 k = 0; k < n; k += m) {
            u64 w = 1;
            for (u32 j = 0; j < m / 2; j++) {
                u64 t = mulmod(w, C[k + j + m / 2], p);
                u64 u = C[k + j];
                C[k + j] = addmod(u, t, p);
                C[k + j + m / 2] = submod(u, t, p);
                w = mulmod(w, wm, p);
            }
        }
    }
    u64 n_inv = invmod(n % p, p), psi_inv = invmod(psi, p), pw = n_inv;
    for (u32 i = 0; i < n; i++) { a[i] = mulmod(C[i], pw, p); pw = mulmod(pw, psi_inv, p); }
    free(B);
    free(C);
}

/* batched: limb b of x (N words) uses prime index idx[b] */
void or_ntt(const or_ctx *c, u64 *x, const u32 *idx, u32 nlimbs) {
#pragma omp parallel for schedule(dynamic)
    for (u32 b = 0; b < nlimbs; b++) ntt_one(x + (size_t)b * c->n, c->log_n, c->m[idx[b]], c->psi[idx[b]]);
}

void or_intt(const or_ctx *c, u64 *x, const u32 *idx, u32 nlimbs) {
#pragma omp parallel for schedule(dynamic)
    for (u32 b = 0; b < nlimbs; b++) intt_one(x + (size_t)b * c->n, c->log_n, c->m[idx[b]], c->psi[idx[b]]);
}

/* The definition itself, one output at a time: ahat[j] = a(psi^(2brv(j)+1)) by Horner. */
void or_ntt_def(const or_ctx *c, const u64 *a, u32 pidx, const u32 *js, u32 nj, u64 *out) {
    u64 p = c->m[pidx];
#pragma omp parallel for
    for (u32 t = 0; t < nj; t++) {
        u64 x = powmod(c->psi[pidx], 2 * (u64)brv(js[t], c->log_n) + 1, p);
        u64 acc = 0;
        for (u32 i = c->n; i-- > 0;) acc = addmod(mulmod(acc, x, p), a[i] % p, p);
        out[t] = acc;
    }
}

/* ---------------------------------------------------------------- elementwise helpers (keygen/decrypt) */

void or_add(const or_ctx *c, const u64 *a, const u64 *b, const u32 *idx, u32 nl, u64 *out) {
    for (u32 l = 0; l < nl; l++)
        for (u32 i = 0; i < c->n; i++) {
            size_t o = (size_t)l * c->n + i;
            out[o] = addmod(a[o], b[o], c->m[idx[l]]);
        }
}

void or_sub(const or_ctx *c, const u64 *a, const u64 *b, const u32 *idx, u32 nl, u64 *out) {
    for (u32 l = 0; l < nl; l++)
        for (u32 i = 0; i < c->n; i++) {
            size_t o = (size_t)l * c->n + i;
            out[o] = submod(a[o], b[o], c->m[idx[l]]);
        }
}

void or_mul(const or_ctx *c, const u64 *a, const u64 *b, const u32 *idx, u32 nl, u64 *out) {
#pragma omp parallel for
    for (u32 l = 0; l < nl; l++)
        for (u32 i = 0; i < c->n; i++) {
            size_t o = (size_t)l * c->n + i;
            out[o] = mulmod(a[o], b[o], c->m[idx[l]]);
        }
}

/* signed integer coefficients -> residues mod each prime (COEFF form) */
void or_lift(const or_ctx *c, const i64 *coef, const u32 *idx, u32 nl, u64 *out) {
    for (u32 l = 0; l < nl; l++) {
        u64 p = c->m[idx[l]];
        for (u32 i = 0; i < c->n; i++) {
            i64 v = coef[i];
            u64 r = v >= 0 ? (u64)v % p : (p - ((u64)(-(v + 1)) + 1) % p) % p;
            out[(size_t)l * c->n + i] = r;
        }
    }
}

/* ---------------------------------------------------------------- automorphism */

/* COEFF form: X^i -> X^(ik mod 2N), negated when ik mod 2N >= N. */
void or_automorph_coeff(const or_ctx *c, const u64 *in, const u32 *idx, u32 nl, u64 galois, u64 *out) {
    u64 two_n = 2 * (u64)c->n;
    for (u32 l = 0; l < nl; l++) {
        u64 p = c->m[idx[l]];
        for (u32 i = 0; i < c->n; i++) {
            u64 e = (u64)i * galois % two_n;
            u64 v = in[(size_t)l * c->n + i];
            if (e >= c->n) out[(size_t)l * c->n + (e - c->n)] = submod(0, v, p);
            else out[(size_t)l * c->n + e] = v;
        }
    }
}

/* EVAL form (SURVEY.md §8(c) reading 15): pi_k(ahat)[j] = ahat[j'] with
 * 2brv(j')+1 = k(2brv(j)+1) mod 2N.  Pure permutation, no sign. */
static u32 eval_src_index(u32 log_n, u32 j, u64 galois) {
    u64 two_n = 2ull << log_n;
    u64 e = (galois % two_n) * (2 * (u64)brv(j, log_n) + 1) % two_n;
    return brv((u32)((e - 1) / 2), log_n);
}

void or_automorph(const or_ctx *c, const u64 *in, u32 nl, u64 galois, u64 *out) {
    for (u32 l = 0; l < nl; l++)
        for (u32 j = 0; j < c->n; j++)
            out[(size_t)l * c->n + j] = in[(size_t)l * c->n + eval_src_index(c->log_n, j, galois)];
}

/* ---------------------------------------------------------------- base conversion (Eq. 1) */

/* PAPER.md:287-322 §3.6.3 eq:conv; SURVEY.md §8(c) readings 13 and 16:
 *   y_i    = [x_i * qhat_i^-1]_{q_i}            (canonical)
 *   out_t  = [ sum_i y_i * [qhat_i]_t ]_t        qhat_i = prod_{m in src, m != i} q_m
 * x: [nsrc][N] COEFF, src/dst: prime indices, out: [ndst][N] COEFF. */
void or_bconv(const or_ctx *c, const u64 *x, const u32 *src, u32 nsrc, const u32 *dst, u32 ndst, u64 *out) {
    u64 *qhat_inv = (u64 *)malloc(sizeof(u64) * nsrc);
    u64 *mat = (u64 *)malloc(sizeof(u64) * nsrc * (ndst ? ndst : 1));
    for (u32 i = 0; i < nsrc; i++) {
        u64 qi = c->m[src[i]], h = 1 % qi;
        for (u32 m = 0; m < nsrc; m++)
            if (m != i) h = mulmod(h, c->m[src[m]] % qi, qi);
        qhat_inv[i] = invmod(h, qi);
        for (u32 t = 0; t < ndst; t++) {
            u64 mt = c->m[dst[t]], v = 1 % mt;
            for (u32 m = 0; m < nsrc; m++)
                if (m != i) v = mulmod(v, c->m[src[m]] % mt, mt);
            mat[(size_t)i * ndst + t] = v;
        }
    }
#pragma omp parallel for schedule(static)
    for (u32 n = 0; n < c->n; n++) {
        u64 y[64];
        for (u32 i = 0; i < nsrc; i++) y[i] = mulmod(x[(size_t)i * c->n + n], qhat_inv[i], c->m[src[i]]);
        for (u32 t = 0; t < ndst; t++) {
            u64 mt = c->m[dst[t]], acc = 0;
            for (u32 i = 0; i < nsrc; i++) acc = addmod(acc, mulmod(y[i], mat[(size_t)i * ndst + t], mt), mt);
            out[(size_t)t * c->n + n] = acc;
        }
    }
    free(qhat_inv);
    free(mat);
}

/* ---------------------------------------------------------------- ModUp */

/* SURVEY.md §8(c) oracle steps 2-3; PAPER.md:288, 318 (§3.6.3).
 * d: [l+1][N] EVAL.  ext: [beta][l+1+K][N] EVAL.  For digit j the limbs of the digit are
 * the input limbs unchanged (EVAL), every other limb t in (Q_l \ digit j) u P is
 * NTT(BConv_{digit j -> t}(INTT(d[digit j]))). */
void or_modup(const or_ctx *c, const u64 *d, u32 level, u64 *ext) {
    u32 n = c->n, ne = level + 1 + c->np, beta = beta_of(c, level);
    u64 *coef = (u64 *)malloc(sizeof(u64) * (size_t)(level + 1) * n);
    u32 *idx = (u32 *)malloc(sizeof(u32) * ne);
    memcpy(coef, d, sizeof(u64) * (size_t)(level + 1) * n);
    for (u32 i = 0; i <= level; i++) idx[i] = i;
    or_intt(c, coef, idx, level + 1);
    for (u32 j = 0; j < beta; j++) {
        u32 lo, hi;
        digit_range(c, level, j, &lo, &hi);
        u64 *Dj = ext + (size_t)j * ne * n;
        u32 nsrc = hi - lo, ndst = 0;
        u32 *src = (u32 *)malloc(sizeof(u32) * nsrc), *dst = (u32 *)malloc(sizeof(u32) * ne);
        u32 *dpos = (u32 *)malloc(sizeof(u32) * ne);
        for (u32 i = 0; i < nsrc; i++) src[i] = lo + i;
        for (u32 t = 0; t < ne; t++) {
            if (t >= lo && t < hi) continue;
            dst[ndst] = ext_prime(c, level, t);
            dpos[ndst++] = t;
        }
        u64 *conv = (u64 *)malloc(sizeof(u64) * (size_t)ndst * n);
        or_bconv(c, coef + (size_t)lo * n, src, nsrc, dst, ndst, conv);
        or_ntt(c, conv, dst, ndst);
        for (u32 u = 0; u < ndst; u++) memcpy(Dj + (size_t)dpos[u] * n, conv + (size_t)u * n, sizeof(u64) * n);
        for (u32 t = lo; t < hi; t++) memcpy(Dj + (size_t)t * n, d + (size_t)t * n, sizeof(u64) * n);
        free(conv); free(src); free(dst); free(dpos);
    }
    free(coef);
    free(idx);
}

/* ---------------------------------------------------------------- key inner product */

/* SURVEY.md §8(c) steps 4-5; PAPER.md:351-352 (§3.6.5 HMult / dot-product fusion):
 *   acc_0[t] = sum_j D_j[t] * b_j[key(t)],  acc_1[t] = sum_j D_j[t] * a_j[key(t)]   (mod t)
 * key(t) = t for Q limbs, L+1+k for P_k.  evk layout [dnum][2][L+1+K][N] with (b, a).
 * galois != 1: D_j[t] <- pi_k(D_j[t]) first (hoisted order, reading 14). */
void or_kip(const or_ctx *c, const u64 *ext, const u64 *evk, u32 level, u64 galois, u64 *acc) {
    u32 n = c->n, ne = level + 1 + c->np, nk = c->nq + c->np, beta = beta_of(c, level);
#pragma omp parallel for schedule(dynamic)
    for (u32 t = 0; t < ne; t++) {
        u32 pi = ext_prime(c, level, t);
        u32 kt = t <= level ? t : c->nq + (t - level - 1);
        u64 p = c->m[pi];
        u64 *tmp = (u64 *)malloc(sizeof(u64) * n);
        u64 *a0 = acc + (size_t)t * n, *a1 = acc + ((size_t)ne + t) * n;
        for (u32 i = 0; i < n; i++) { a0[i] = 0; a1[i] = 0; }
        for (u32 j = 0; j < beta; j++) {
            const u64 *D = ext + ((size_t)j * ne + t) * n;
            if (galois != 1) { or_automorph(c, D, 1, galois, tmp); D = tmp; }
            const u64 *bj = evk + (((size_t)j * 2 + 0) * nk + kt) * n;
            const u64 *aj = evk + (((size_t)j * 2 + 1) * nk + kt) * n;
            for (u32 i = 0; i < n; i++) {
                a0[i] = addmod(a0[i], mulmod(D[i], bj[i], p), p);
                a1[i] = addmod(a1[i], mulmod(D[i], aj[i], p), p);
            }
        }
        free(tmp);
    }
}

/* ---------------------------------------------------------------- ModDown */

/* SURVEY.md §8(c) step 6; PAPER.md:288, 350 (§3.6.5 ModDown fusion "P^-1(x - NTT(x'))");
 * SPEC.md:470-477.  acc: [l+1+K][N] EVAL -> out: [l+1][N] EVAL.
 *   y = INTT(acc[P]);  conv = BConv_{P -> Q_l}(y);  out_i = (acc_i - NTT(conv)_i) * P^-1 mod q_i */
void or_moddown(const or_ctx *c, const u64 *acc, u32 level, u64 *out) {
    u32 n = c->n, K = c->np;
    u64 *pc = (u64 *)malloc(sizeof(u64) * (size_t)K * n);
    u64 *conv = (u64 *)malloc(sizeof(u64) * (size_t)(level + 1) * n);
    u32 *pidx = (u32 *)malloc(sizeof(u32) * K), *qidx = (u32 *)malloc(sizeof(u32) * (level + 1));
    for (u32 k = 0; k < K; k++) pidx[k] = c->nq + k;
    for (u32 i = 0; i <= level; i++) qidx[i] = i;
    memcpy(pc, acc + (size_t)(level + 1) * n, sizeof(u64) * (size_t)K * n);
    or_intt(c, pc, pidx, K);
    or_bconv(c, pc, pidx, K, qidx, level + 1, conv);
    or_ntt(c, conv, qidx, level + 1);
    for (u32 i = 0; i <= level; i++) {
        u64 q = c->m[i], P = 1;
        for (u32 k = 0; k < K; k++) P = mulmod(P, c->m[c->nq + k] % q, q);
        u64 Pinv = invmod(P, q);
        for (u32 x = 0; x < n; x++) {
            size_t o = (size_t)i * n + x;
            out[o] = mulmod(submod(acc[o], conv[o], q), Pinv, q);
        }
    }
    free(pc); free(conv); free(pidx); free(qidx);
}

/* ---------------------------------------------------------------- KeySwitch, rotations */

/* KeySwitch(c0, c1) = (c0 + ModDown(acc0), ModDown(acc1)). */
static void ks_from_ext(const or_ctx *c, const u64 *c0, const u64 *ext, u32 level, const u64 *evk,
                        u64 galois, u64 *out0, u64 *out1) {
    u32 n = c->n, ne = level + 1 + c->np;
    u64 *acc = (u64 *)malloc(sizeof(u64) * (size_t)2 * ne * n);
    u64 *md = (u64 *)malloc(sizeof(u64) * (size_t)(level + 1) * n);
    u32 *qidx = (u32 *)malloc(sizeof(u32) * (level + 1));
    for (u32 i = 0; i <= level; i++) qidx[i] = i;
    or_kip(c, ext, evk, level, galois, acc);
    or_moddown(c, acc, level, md);
    or_add(c, c0, md, qidx, level + 1, out0);
    or_moddown(c, acc + (size_t)ne * n, level, out1);
    free(acc); free(md); free(qidx);
}

void or_keyswitch(const or_ctx *c, const u64 *c0, const u64 *c1, u32 level, const u64 *evk, u64 *out0, u64 *out1) {
    size_t sz = (size_t)beta_of(c, level) * (level + 1 + c->np) * c->n;
    u64 *ext = (u64 *)malloc(sizeof(u64) * sz);
    or_modup(c, c1, level, ext);
    ks_from_ext(c, c0, ext, level, evk, 1, out0, out1);
    free(ext);
}

/* Hoisted rotations (§3.6.6; SURVEY.md reading 14): one ModUp of c1, then
 * per rotation r: D_j <- pi_k(D_j) inside the key inner product, ModDown, and
 * out0 = pi_k(c0) + ModDown(acc0), out1 = ModDown(acc1). */
void or_rotate_hoisted(const or_ctx *c, const u64 *c0, const u64 *c1, u32 level, u32 nrot, const u64 *galois,
                       const u64 *const *evk, u64 *const *out0, u64 *const *out1) {
    size_t sz = (size_t)beta_of(c, level) * (level + 1 + c->np) * c->n;
    u64 *ext = (u64 *)malloc(sizeof(u64) * sz);
    u64 *rc0 = (u64 *)malloc(sizeof(u64) * (size_t)(level + 1) * c->n);
    or_modup(c, c1, level, ext);
    for (u32 r = 0; r < nrot; r++) {
        or_automorph(c, c0, level + 1, galois[r], rc0);
        ks_from_ext(c, rc0, ext, level, evk[r], galois[r], out0[r], out1[r]);
    }
    free(ext);
    free(rc0);
}

/* Unhoisted rotation: KeySwitch(pi_k(c0), pi_k(c1)) -- used only for decrypt-level checks. */
void or_rotate(const or_ctx *c, const u64 *c0, const u64 *c1, u32 level, u64 galois, const u64 *evk,
               u64 *out0, u64 *out1) {
    size_t sz = (size_t)(level + 1) * c->n;
    u64 *r0 = (u64 *)malloc(sizeof(u64) * sz), *r1 = (u64 *)malloc(sizeof(u64) * sz);
    or_automorph(c, c0, level + 1, galois, r0);
    or_automorph(c, c1, level + 1, galois, r1);
    or_keyswitch(c, r0, r1, level, evk, out0, out1);
    free(r0);
    free(r1);
}

/* ---------------------------------------------------------------- HMult front-end, Rescale */

/* Tensor product of two ciphertexts in EVAL form (§3.6.5 HMult fusion lists its
 * three outputs c0*c0', c0*c1' + c1*c0', c1*c1'; "tensor product (c0c0', c0c1'+c1c0',
 * c1c1')"):  d0 = a0*b0, d1 = a0*b1 + a1*b0, d2 = a1*b1 (mod q_i), limbs 0..l. */
void or_tensor(const or_ctx *c, const u64 *a0, const u64 *a1, const u64 *b0, const u64 *b1, u32 level,
               u64 *d0, u64 *d1, u64 *d2) {
    u32 n = c->n;
    for (u32 i = 0; i <= level; i++) {
        u64 q = c->m[i];
        for (u32 x = 0; x < n; x++) {
            size_t o = (size_t)i * n + x;
            d0[o] = mulmod(a0[o], b0[o], q);
            d1[o] = addmod(mulmod(a0[o], b1[o], q), mulmod(a1[o], b0[o], q), q);
            d2[o] = mulmod(a1[o], b1[o], q);
        }
    }
}

/* HMult without rescale (Table 1 "HMult"): tensor product, then
 * relinearisation of d2 by hybrid key switching with the relinearisation key:
 *   out0 = d0 + ModDown(acc0), out1 = d1 + ModDown(acc1),  acc = KIP(ModUp(d2)). */
void or_hmult(const or_ctx *c, const u64 *a0, const u64 *a1, const u64 *b0, const u64 *b1, u32 level,
              const u64 *evk, u64 *out0, u64 *out1) {
    size_t sz = (size_t)(level + 1) * c->n;
    u64 *d0 = (u64 *)malloc(sizeof(u64) * sz), *d1 = (u64 *)malloc(sizeof(u64) * sz);
    u64 *d2 = (u64 *)malloc(sizeof(u64) * sz), *t1 = (u64 *)malloc(sizeof(u64) * sz);
    u32 *qidx = (u32 *)malloc(sizeof(u32) * (level + 1));
    for (u32 i = 0; i <= level; i++) qidx[i] = i;
    or_tensor(c, a0, a1, b0, b1, level, d0, d1, d2);
    or_keyswitch(c, d0, d2, level, evk, out0, t1);
    or_add(c, d1, t1, qidx, level + 1, out1);
    free(d0); free(d1); free(d2); free(t1); free(qidx);
}

/* Rescale of one polynomial x [l+1][N] EVAL at level l >= 1 to level l-1 (Table 1
 * "Rescale after multiplication"; §3.6.5 "q_l^{-1}(x^{(i)} - NTT(SwitchModulo(x^{(l)})))"):
 *   t    = INTT_{q_l}(x_l)                                   (COEFF, [0, q_l))
 *   s_i  = SwitchModulo(t) into q_i, centered: t if 2t < q_l, else t - q_l   (reading 15)
 *   out_i = q_l^{-1} (x_i - NTT_{q_i}(s_i)) mod q_i,  i < l.
 * Centered SwitchModulo makes the result the rounded quotient round(X / q_l) of the CRT value X. */
void or_rescale(const or_ctx *c, const u64 *x, u32 level, u64 *out) {
    u32 n = c->n;
    u64 ql = c->m[level];
    u64 *t = (u64 *)malloc(sizeof(u64) * n), *s = (u64 *)malloc(sizeof(u64) * n);
    u32 li = level;
    memcpy(t, x + (size_t)level * n, sizeof(u64) * n);
    or_intt(c, t, &li, 1);
    for (u32 i = 0; i < level; i++) {
        u64 q = c->m[i];
        for (u32 k = 0; k < n; k++) {
            if ((u128)t[k] * 2 < ql) s[k] = t[k] % q;
            else s[k] = submod(t[k] % q, ql % q, q); /* t - q_l (negative) mod q */
        }
        or_ntt(c, s, &i, 1);
        u64 qinv = invmod(ql % q, q);
        for (u32 k = 0; k < n; k++) {
            size_t o = (size_t)i * n + k;
            out[o] = mulmod(submod(x[o], s[k], q), qinv, q);
        }
    }
    free(t);
    free(s);
}

/* ---------------------------------------------------------------- BSGS linear transform (NEXT-2) */

/* Fused plaintext-weighted sum of ciphertexts (§3.6.5 "a weighed sum can be reduced
 * from 4n-2 down to n+1 memory operations"): out_p = sum_j w_j * x_{j,p} (mod q_i), p = 0, 1.
 * x0[j], x1[j], w[j]: [l+1][N] EVAL. */
void or_pt_wsum(const or_ctx *c, u32 nterm, const u64 *const *w, const u64 *const *x0, const u64 *const *x1,
                u32 level, u64 *out0, u64 *out1) {
    u32 n = c->n;
    for (u32 i = 0; i <= level; i++) {
        u64 q = c->m[i];
        for (u32 k = 0; k < n; k++) {
            size_t o = (size_t)i * n + k;
            u64 s0 = 0, s1 = 0;
            for (u32 j = 0; j < nterm; j++) {
                s0 = addmod(s0, mulmod(w[j][o], x0[j][o], q), q);
                s1 = addmod(s1, mulmod(w[j][o], x1[j][o], q), q);
            }
            out0[o] = s0;
            out1[o] = s1;
        }
    }
}

/* Ciphertext x plaintext-matrix product by baby-step giant-step (§3.6.7: "Each
 * ciphertext-vector times plaintext-matrix multiplication is then performed using a BSGS algorithm,
 * which reduces the number of required rotations and leverages the hoisted rotation optimization";
 * no ModDown hoisting; SPEC.md:576-583 homomorphic_linear_transform):
 *   ct_0 = ct, ct_j = RotHoisted_{bg[j-1]}(ct) for j = 1..n1-1 (one shared ModUp);
 *   I_i  = sum_j pt[i*n1 + j] * ct_j  (i < n2);
 *   out  = I_0 + sum_{i>=1} RotHoisted_{gg[i-1]}(I_i)  (one rotation per giant step).
 * pt[i*n1+j] [l+1][N] EVAL are the (pre-rotated) diagonals; bk[j-1], gk[i-1] the rotation keys. */
void or_lintrans(const or_ctx *c, const u64 *c0, const u64 *c1, u32 level, u32 n1, u32 n2, const u64 *bg,
                 const u64 *const *bk, const u64 *gg, const u64 *const *gk, const u64 *const *pt, u64 *out0,
                 u64 *out1) {
    size_t sz = (size_t)(level + 1) * c->n;
    u64 **b0 = (u64 **)malloc(sizeof(u64 *) * n1), **b1 = (u64 **)malloc(sizeof(u64 *) * n1);
    b0[0] = (u64 *)c0;
    b1[0] = (u64 *)c1;
    for (u32 j = 1; j < n1; j++) {
        b0[j] = (u64 *)malloc(sizeof(u64) * sz);
        b1[j] = (u64 *)malloc(sizeof(u64) * sz);
    }
    if (n1 > 1) or_rotate_hoisted(c, c0, c1, level, n1 - 1, bg, bk, b0 + 1, b1 + 1);
    u64 *i0 = (u64 *)malloc(sizeof(u64) * sz), *i1 = (u64 *)malloc(sizeof(u64) * sz);
    u64 *r0 = (u64 *)malloc(sizeof(u64) * sz), *r1 = (u64 *)malloc(sizeof(u64) * sz);
    u32 *qidx = (u32 *)malloc(sizeof(u32) * (level + 1));
    for (u32 i = 0; i <= level; i++) qidx[i] = i;
    for (u32 i = 0; i < n2; i++) {
        or_pt_wsum(c, n1, pt + (size_t)i * n1, (const u64 *const *)b0, (const u64 *const *)b1, level, i0, i1);
        if (i == 0) {
            memcpy(out0, i0, sizeof(u64) * sz);
            memcpy(out1, i1, sizeof(u64) * sz);
        } else {
            or_rotate_hoisted(c, i0, i1, level, 1, gg + (i - 1), gk + (i - 1), &r0, &r1);
            or_add(c, out0, r0, qidx, level + 1, out0);
            or_add(c, out1, r1, qidx, level + 1, out1);
        }
    }
    for (u32 j = 1; j < n1; j++) {
        free(b0[j]);
        free(b1[j]);
    }
    free(b0); free(b1); free(i0); free(i1); free(r0); free(r1); free(qidx);
}

/* ---------------------------------------------------------------- client side (harness only) */

/* Key-switching key generation (SURVEY.md §8(c) "oracle-side keygen", reading 10):
 *   evk_j = (b_j, a_j) over all L+1+K limbs, b_j = -a_j*s + e_j + P*Qtilde_j*s_old,
 * Qtilde_j = CRT idempotent of digit j at level L (1 mod q_i in digit j, 0 mod other q,
 * and P*Qtilde_j = 0 mod every p_k).  Inputs: s_eval / s_old_eval [L+1+K][N] EVAL,
 * a [dnum][L+1+K][N] EVAL uniform, e [dnum][N] signed COEFF.  Output evk [dnum][2][L+1+K][N]. */
void or_keygen_ks(const or_ctx *c, const u64 *s_eval, const u64 *s_old_eval, const u64 *a, const i64 *e, u64 *evk) {
    u32 n = c->n, nk = c->nq + c->np;
    u32 *idx = (u32 *)malloc(sizeof(u32) * nk);
    for (u32 i = 0; i < nk; i++) idx[i] = i;
    u64 *ee = (u64 *)malloc(sizeof(u64) * (size_t)nk * n);
    for (u32 j = 0; j < c->dnum; j++) {
        or_lift(c, e + (size_t)j * n, idx, nk, ee);
        or_ntt(c, ee, idx, nk);
        u64 *b = evk + ((size_t)j * 2 + 0) * nk * n, *aa = evk + ((size_t)j * 2 + 1) * nk * n;
        const u64 *aj = a + (size_t)j * nk * n;
        memcpy(aa, aj, sizeof(u64) * (size_t)nk * n);
        u32 lo = j * c->alpha, hi = (j + 1) * c->alpha < c->nq ? (j + 1) * c->alpha : c->nq;
        for (u32 l = 0; l < nk; l++) {
            u64 p = c->m[l], Pm = 1;
            for (u32 k = 0; k < c->np; k++) Pm = mulmod(Pm, c->m[c->nq + k] % p, p);
            u64 g = (l >= lo && l < hi) ? Pm : 0; /* P*Qtilde_j mod m_l */
            for (u32 x = 0; x < n; x++) {
                size_t o = (size_t)l * n + x;
                u64 v = submod(ee[o], mulmod(aj[o], s_eval[o], p), p);
                b[o] = addmod(v, mulmod(g, s_old_eval[o], p), p);
            }
        }
    }
    free(idx);
    free(ee);
}

/* Decryption to COEFF residues: m_i = INTT(c0 + c1*s) on limbs 0..l. */
void or_decrypt(const or_ctx *c, const u64 *c0, const u64 *c1, u32 level, const u64 *s_eval, u64 *out) {
    u32 *idx = (u32 *)malloc(sizeof(u32) * (level + 1));
    for (u32 i = 0; i <= level; i++) idx[i] = i;
    u64 *t = (u64 *)malloc(sizeof(u64) * (size_t)(level + 1) * c->n);
    or_mul(c, c1, s_eval, idx, level + 1, t);
    or_add(c, c0, t, idx, level + 1, out);
    or_intt(c, out, idx, level + 1);
    free(idx);
    free(t);
}
