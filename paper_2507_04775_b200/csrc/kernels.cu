// kernels.cu -- base conversion (Eq. 1), evaluation-key inner product, EVAL automorphism, and the
// tensor-core column pass of the NTT (opt-in).
//
// All are cross-limb, same-coefficient passes (§3.6.1 dependency classes).  The base
// conversion is, across the N coefficients, a dense contraction with a constant matrix, and runs on the
// tcgen05 tensor cores through an exact byte-split identity (k_bconv_tc); the warp-level
// IMMA and the integer-pipe kernels (30-bit-split IMAD.WIDE MACs, "128-bit accumulation, one reduction
// per output") remain behind switches and are tested for identical bits.  The key inner
// product is element-wise (no shared operand) and stays on the integer pipe.
#include <stdlib.h>

#include "internal.h"
#include "tc.cuh"

// source limb i of a base-conversion group: an absolute (possibly peer-mapped) address, or a slot of A.in
__device__ __forceinline__ const u64 *bc_src(const BconvArgs &A, const BconvGroup &G, int i, size_t N) {
    return G.srcp[i] ? G.srcp[i] : A.in + (size_t)G.src_slot[i] * N;
}

// ------------------------------------------------------------------------------------------------
// Base conversion (§3.6.3, eq:conv):  out_t = [ sum_i y_i [qhat_i]_t ]_t.
// grid.x: coefficient blocks (2 coefficients / thread), grid.y: group (digit or polynomial).
// grid.x: coefficient blocks (2 coefficients / thread), grid.y: group (digit or polynomial),
// grid.z: chunk of BC_TCH targets.  LAZY: outputs in [0, 8t) for a consumer that accepts the lazy
// range (the forward NTT); otherwise canonical.
#ifndef HKS_BC_TCH
#define HKS_BC_TCH 10
#endif
#define BC_TCH HKS_BC_TCH
template <int NSRC, bool LAZY, int CPT>
__global__ void __launch_bounds__(256, (CPT == 1 && NSRC <= 10) ? 5 : 3) k_bconv(const __grid_constant__ BconvArgs A) {
    pdl_trigger();
    pdl_wait();
    const BconvGroup &G = A.g[blockIdx.y];
    const u32 u0 = blockIdx.z * BC_TCH;
    if (u0 >= G.ndst) return;
    const u32 nt = min((u32)BC_TCH, G.ndst - u0);
    __shared__ uint2 smat[NSRC * BC_TCH];
    __shared__ PrimeConst spc[BC_TCH];
    for (u32 idx = threadIdx.x; idx < NSRC * nt; idx += blockDim.x) {
        const u32 i = idx / nt, u = idx - i * nt;
        smat[i * BC_TCH + u] = G.mat[(size_t)i * G.mat_stride + u0 + u];
    }
    for (u32 u = threadIdx.x; u < nt; u += blockDim.x) spc[u] = A.pc[G.dst_prime[u0 + u]];
    __syncthreads();

    const size_t N = (size_t)1 << A.log_n;
    const size_t x0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * CPT;
    if (x0 >= N) return;
    u32 yl[NSRC][CPT], yh[NSRC][CPT];
#pragma unroll
    for (int i = 0; i < NSRC; i++) {
        u64 v[CPT];
        if (CPT == 2) {
            const ulonglong2 t = *reinterpret_cast<const ulonglong2 *>(bc_src(A, G, i, N) + x0);
            v[0] = t.x;
            v[CPT - 1] = t.y;
        } else {
            v[0] = bc_src(A, G, i, N)[x0];
        }
#pragma unroll
        for (int c = 0; c < CPT; c++) split30(v[c], yl[i][c], yh[i][c]);
    }
    for (u32 u = 0; u < nt; u++) {
        Acc30 a[CPT];
        {
            const uint2 m = smat[u];
#pragma unroll
            for (int c = 0; c < CPT; c++) acc_first(a[c], yl[0][c], yh[0][c], m.x, m.y);
        }
#pragma unroll
        for (int i = 1; i < NSRC; i++) {
            const uint2 m = smat[i * BC_TCH + u];
#pragma unroll
            for (int c = 0; c < CPT; c++) acc_mac(a[c], yl[i][c], yh[i][c], m.x, m.y);
        }
        const PrimeConst pc = spc[u];
        u64 o[CPT];
#pragma unroll
        for (int c = 0; c < CPT; c++) o[c] = LAZY ? acc_reduce_lazy(a[c], pc) : acc_reduce(a[c], pc);
        u64 *dst = A.out + (size_t)G.dst_slot[u0 + u] * N + x0;
        if (CPT == 2)
            *reinterpret_cast<ulonglong2 *>(dst) = make_ulonglong2(o[0], o[CPT - 1]);
        else
            dst[0] = o[0];
    }
}

// Karatsuba variant (3 IMAD.WIDE per MAC instead of 4), one coefficient per thread, NSRC <= 11.
template <int NSRC, bool LAZY>
__global__ void __launch_bounds__(256, 3) k_bconv_kara(const __grid_constant__ BconvArgs A) {
    pdl_trigger();
    const BconvGroup &G = A.g[blockIdx.y];
    const u32 u0 = blockIdx.z * BC_TCH;
    if (u0 >= G.ndst) return;
    const u32 nt = min((u32)BC_TCH, G.ndst - u0);
    __shared__ uint4 smat[NSRC * BC_TCH];
    __shared__ PrimeConst spc[BC_TCH];
    for (u32 idx = threadIdx.x; idx < NSRC * nt; idx += blockDim.x) {
        const u32 i = idx / nt, u = idx - i * nt;
        const uint2 m = G.mat[(size_t)i * G.mat_stride + u0 + u];
        smat[i * BC_TCH + u] = make_uint4(m.x, m.y, G.mats[(size_t)i * G.mat_stride + u0 + u], 0);
    }
    for (u32 u = threadIdx.x; u < nt; u += blockDim.x) spc[u] = A.pc[G.dst_prime[u0 + u]];
    __syncthreads();
    pdl_wait();   // ctx tables above are immutable; the inputs below come from the predecessor

    const size_t N = (size_t)1 << A.log_n;
    const size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= N) return;
    u32 yl[NSRC], yh[NSRC];
#pragma unroll
    for (int i = 0; i < NSRC; i++) split30(bc_src(A, G, i, N)[x], yl[i], yh[i]);
    // two targets per iteration: their independent MAC/reduction chains interleave
    for (u32 u = 0; u < nt; u += 2) {
        const u32 v = (u + 1 < nt) ? u + 1 : u;
        AccK a, b;
#define KMAC(I) if (I < NSRC) { const uint4 m = smat[I * BC_TCH + u], mb = smat[I * BC_TCH + v]; \
        const u32 ys = yl[I] + yh[I]; acck_mac<I>(a, yl[I], yh[I], ys, m.x, m.y, m.z); acck_mac<I>(b, yl[I], yh[I], ys, mb.x, mb.y, mb.z); }
        KMAC(0) KMAC(1) KMAC(2) KMAC(3) KMAC(4) KMAC(5) KMAC(6) KMAC(7) KMAC(8) KMAC(9) KMAC(10) KMAC(11)
#undef KMAC
        u64 lo, hi, lob, hib;
        acck_to128(a, NSRC, lo, hi);
        acck_to128(b, NSRC, lob, hib);
        const PrimeConst pc = spc[u], pcb = spc[v];
        const u64 ra = LAZY ? reduce128_lazy(lo, hi, pc) : reduce128(lo, hi, pc);
        const u64 rb = LAZY ? reduce128_lazy(lob, hib, pcb) : reduce128(lob, hib, pcb);
        A.out[(size_t)G.dst_slot[u0 + u] * N + x] = ra;
        if (v != u) A.out[(size_t)G.dst_slot[u0 + v] * N + x] = rb;
    }
}

template <int NSRC>
static void bconv_kara_go(const BconvArgs &a, cudaStream_t s) {
    const u32 threads = 256;
    const size_t N = (size_t)1 << a.log_n;
    u32 maxdst = 0;
    for (u32 g = 0; g < a.ngroups; g++) maxdst = max(maxdst, a.g[g].ndst);
    dim3 grid((u32)((N + threads - 1) / threads), a.ngroups, (maxdst + BC_TCH - 1) / BC_TCH);
    ProfScope ps(K_BCONV, s);
    if (a.lazy_out)
        (void)hks_launch(k_bconv_kara<NSRC, true>, grid, dim3(threads), 0, s, a);
    else
        (void)hks_launch(k_bconv_kara<NSRC, false>, grid, dim3(threads), 0, s, a);
    double words = 0, macs = 0;
    for (u32 g = 0; g < a.ngroups; g++) {
        words += a.g[g].nsrc + a.g[g].ndst;
        macs += (double)a.g[g].nsrc * a.g[g].ndst;
    }
    ps.done(words * (double)N * 8.0, macs * (double)N * 4.0);
}

#if HKS_EXPERIMENTAL
// ------------------------------------------------------------------------------------------------
// Base conversion on the tensor pipe.  Eq. 1 is, across the N coefficients, a dense contraction
// OUT[t][x] = sum_i M[i][t] Y[i][x] with a constant matrix.  Splitting y_i into bytes y_{i,a} and
// folding the byte weight into the matrix, m_{i,t,a} = 2^(8a) M[i][t] mod t, gives an exact integer
// identity   X'_t(x) = sum_c 2^(8c) S_{t,c}(x),  S_{t,c}(x) = sum_{i,a} y_{i,a}(x) byte_c(m_{i,t,a}),
// with X' == sum_i y_i M[i][t] (mod t): a u8 x u8 GEMM of K = 8 NSRC and 8 byte columns per target,
// computed with warp-level IMMA (m16n8k32 / m16n8k16, s32 accumulators: S < 128 * 255^2 < 2^23), and
// one 80-bit reduction per output ("reduced only before being written back").  The
// output is congruent to the Eq. 1 value, so canonical outputs are identical to k_bconv's and lazy
// ones ([0, 6t)) differ only inside the forward NTT's accepted input range.
//
// Operands: A = the byte-column matrix (M = 16 rows = 8 targets x 2 byte columns per m-tile, from
// shared memory), B = the input bytes (N = 8 coefficients per n-tile, straight from the limbs), so a
// lane's B fragment of a k32 step is one whole word: lane (g, q) holds y_{4s+q}[x0+g] (bytes 0-3 in b0,
// 4-7 in b1) -- k-step s covers sources 4s..4s+3; a trailing k16 step takes 1-2 sources, lane q holding
// half (q & 1) of y_{4s + q/2}.  Row g (g + 8) of m-tile i is (target g of the warp's block, byte column
// c = 2i (2i + 1)), so after the 4 m-tiles lane (g, q) holds all eight S_{t,c} of target g for the
// coefficients x0 + 2q and x0 + 2q + 1: no shuffles, one 16-byte store per lane and n-tile.
#ifndef HKS_MMA_TCH
#define HKS_MMA_TCH 32
#endif
#ifndef HKS_MMA_CW
#define HKS_MMA_CW 128
#endif
#ifndef HKS_MMA_MINB
#define HKS_MMA_MINB 2
#endif
#ifndef HKS_MMA_NPI
#define HKS_MMA_NPI 2
#endif
#define MMA_TCH HKS_MMA_TCH
#define MMA_CW HKS_MMA_CW
#define NPI HKS_MMA_NPI
template <int NSRC, bool LAZY>
__global__ void __launch_bounds__(256, HKS_MMA_MINB) k_bconv_mma(const __grid_constant__ BconvArgs A) {
    pdl_trigger();
    constexpr int KS32 = NSRC / 4 + (NSRC % 4 == 3 ? 1 : 0);   // k32 steps (the last one may be padded)
    constexpr bool K16 = (NSRC % 4 == 1 || NSRC % 4 == 2);    // trailing k16 step
    constexpr int NS = KS32 + (K16 ? 1 : 0);
    constexpr int NB = MMA_TCH / 8;                            // target blocks (8 targets) per CTA
    const BconvGroup &G = A.g[blockIdx.y];
    const u32 u0 = blockIdx.z * MMA_TCH;
    if (u0 >= G.ndst) return;
    const u32 nt = min((u32)MMA_TCH, G.ndst - u0);
    const u32 nblk = (nt + 7) / 8;
    // A fragments [block][m-tile i][k-step s][lane] as uint4 (a0, a1, a2, a3)
    __shared__ uint4 sA[NB * 4 * NS * 32];
    __shared__ uint2 sA16[K16 ? NB * 4 * 32 : 1];   // k16-step fragments (a0, a1), lane-contiguous
    __shared__ PrimeConst spc[MMA_TCH];
    {
        // all table loads of a thread are issued before its shared-memory stores (one L2 round trip)
        constexpr int PER = (NB * 4 * NS * 32 + 255) / 256;
        const u32 ne = nblk * 4 * NS * 32;
        ulonglong2 w[PER];
#pragma unroll
        for (int r = 0; r < PER; r++) {
            const u32 idx = threadIdx.x + 256 * r;
            const u32 ln = idx & 31, s = (idx >> 5) % NS, mi = (idx >> 5) / NS % 4, tb = (idx >> 5) / NS / 4;
            const u32 g = ln >> 2, q = ln & 3, u = tb * 8 + g;
            const u32 i = (K16 && (int)s == KS32) ? 4 * s + (q >> 1) : 4 * s + q;
            w[r] = make_ulonglong2(0, 0);
            if (idx < ne && u < nt && i < (u32)NSRC)
                w[r] = __ldg(reinterpret_cast<const ulonglong2 *>(G.matb + ((size_t)i * G.mat_stride + u0 + u) * 8 + 2 * mi));
        }
#pragma unroll
        for (int r = 0; r < PER; r++) {
            const u32 idx = threadIdx.x + 256 * r;
            if (idx >= ne) break;
            const u32 ln = idx & 31, s = (idx >> 5) % NS, mi = (idx >> 5) / NS % 4, tb = (idx >> 5) / NS / 4;
            const u32 q = ln & 3;
            if (K16 && (int)s == KS32) {
                const u32 sh = (q & 1) * 32;
                sA16[(tb * 4 + mi) * 32 + ln] = make_uint2((u32)(w[r].x >> sh), (u32)(w[r].y >> sh));
            } else {
                sA[idx] = make_uint4((u32)w[r].x, (u32)w[r].y, (u32)(w[r].x >> 32), (u32)(w[r].y >> 32));
            }
        }
    }
    for (u32 u = threadIdx.x; u < nt; u += blockDim.x) spc[u] = A.pc[G.dst_prime[u0 + u]];
    __syncthreads();
    pdl_wait();   // ctx tables above are immutable; the inputs below come from the predecessor

    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    const u32 nparts = 8 / nblk, tb = warp % nblk, part = warp / nblk;
    if (part >= nparts) return;
    const u32 u = tb * 8 + g;
    const bool active = u < nt;
    const PrimeConst pc = spc[active ? u : 0];
    const size_t N = (size_t)1 << A.log_n;
    u64 *dst = A.out + (size_t)G.dst_slot[u0 + (active ? u : 0)] * N;
    const uint4 *fa = sA + tb * 4 * NS * 32 + lane;
    const uint2 *fa16 = sA16 + (K16 ? tb * 4 * 32 + lane : 0);
    const u64 *src[NS];
#pragma unroll
    for (int s = 0; s < NS; s++) {
        const u32 i = (K16 && s == KS32) ? 4 * s + (q >> 1) : 4 * s + q;
        src[s] = i < (u32)NSRC ? bc_src(A, G, i, N) + g : nullptr;
    }
    const size_t xbeg = (size_t)blockIdx.x * A.cw, xend = xbeg + A.cw, xstep = 8 * NPI * nparts;
    // NPI n-tiles (8 NPI coefficients) per iteration: 4 NPI independent accumulator chains; the next
    // iteration's input words are requested before this one's MMAs (register double buffer)
    u64 ynx[NPI][NS];
#pragma unroll
    for (int s = 0; s < NS; s++)
#pragma unroll
        for (int n = 0; n < NPI; n++) ynx[n][s] = src[s] ? __ldg(src[s] + xbeg + 8 * NPI * part + 8 * n) : 0;
    for (size_t x0 = xbeg + 8 * NPI * part; x0 < xend; x0 += xstep) {
        u64 yb[NPI][NS];
#pragma unroll
        for (int s = 0; s < NS; s++)
#pragma unroll
            for (int n = 0; n < NPI; n++) yb[n][s] = ynx[n][s];
        if (x0 + xstep < xend) {
#pragma unroll
            for (int s = 0; s < NS; s++)
#pragma unroll
                for (int n = 0; n < NPI; n++) ynx[n][s] = src[s] ? __ldg(src[s] + x0 + xstep + 8 * n) : 0;
        }
        int acc[NPI][4][4];
#pragma unroll
        for (int n = 0; n < NPI; n++)
#pragma unroll
            for (int mi = 0; mi < 4; mi++) acc[n][mi][0] = acc[n][mi][1] = acc[n][mi][2] = acc[n][mi][3] = 0;
#pragma unroll
        for (int s = 0; s < NS; s++) {
#pragma unroll
            for (int mi = 0; mi < 4; mi++) {
                if (K16 && s == KS32) {
                    const uint2 a = fa16[mi * 32];
#pragma unroll
                    for (int n = 0; n < NPI; n++) {
                        const u32 b = (q & 1) ? (u32)(yb[n][s] >> 32) : (u32)yb[n][s];
                        mma_u8_k16(acc[n][mi], a.x, a.y, b);
                    }
                } else {
                    const uint4 a = fa[(mi * NS + s) * 32];
                    const u32 af[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                    for (int n = 0; n < NPI; n++) mma_u8_k32(acc[n][mi], af, (u32)yb[n][s], (u32)(yb[n][s] >> 32));
                }
            }
        }
        if (active) {
#pragma unroll
            for (int n = 0; n < NPI; n++) {
                u64 o[2];
#pragma unroll
                for (int e = 0; e < 2; e++)
                    o[e] = bytesum_reduce<LAZY>(acc[n][0][e], acc[n][0][2 + e], acc[n][1][e], acc[n][1][2 + e],
                                                acc[n][2][e], acc[n][2][2 + e], acc[n][3][e], acc[n][3][2 + e], pc);
                *reinterpret_cast<ulonglong2 *>(dst + x0 + 8 * n + 2 * q) = make_ulonglong2(o[0], o[1]);
            }
        }
    }
}

template <int NSRC>
static void bconv_mma_go(const BconvArgs &a, cudaStream_t s) {
    const size_t N = (size_t)1 << a.log_n;
    u32 maxdst = 0;
    for (u32 g = 0; g < a.ngroups; g++) maxdst = max(maxdst, a.g[g].ndst);
    // one wave: every CTA stages its matrix fragments before griddepcontrol.wait, i.e. while the
    // predecessor is still running (MMA_SLOTS resident CTAs per SM); CW = coefficients per CTA
    const u32 nz = (maxdst + MMA_TCH - 1) / MMA_TCH;
    const int nsm = hks_num_sms();
    size_t cw = MMA_CW;
    while (cw < N && (N / cw) * a.ngroups * nz > (size_t)nsm * HKS_MMA_MINB) cw *= 2;
    BconvArgs b = a;
    b.cw = (u32)cw;
    dim3 grid((u32)(N / cw), a.ngroups, nz);
    ProfScope ps(K_BCONV, s);
    if (a.lazy_out)
        (void)hks_launch(k_bconv_mma<NSRC, true>, grid, dim3(256), 0, s, b);
    else
        (void)hks_launch(k_bconv_mma<NSRC, false>, grid, dim3(256), 0, s, b);
    double words = 0, macs = 0;
    for (u32 g = 0; g < a.ngroups; g++) {
        words += a.g[g].nsrc + a.g[g].ndst;
        macs += (double)a.g[g].nsrc * a.g[g].ndst;
    }
    (void)macs;   // the contraction runs on the tensor pipe (IMMA): no integer-pipe products to count
    ps.done(words * (double)N * 8.0, 0.0);
}

#endif  // HKS_EXPERIMENTAL

// ------------------------------------------------------------------------------------------------
// The same byte-split contraction on the 5th-generation tensor cores (tcgen05, accumulators in TMEM).
//   D[m][8t + c] (s32, TMEM lane m, column 8t + c) = sum_k A[m][k] B[8t + c][k]
//   A = input tile: 128 coefficients x K bytes (source i, byte a) -- K-major, no swizzle: core
//       matrices of 8 rows x 16 bytes, the 16 bytes of row m / chunk kc being y_{2kc}[x_m], y_{2kc+1}[x_m]
//   B = byte-column matrix: row 8t + c, chunk kc = matb words (2kc, t, c), (2kc + 1, t, c)
// so TMEM lane m holds, in 8 consecutive columns, the eight S_{t,c} of coefficient m and target t:
// one tcgen05.ld (32x32b.x8) per output.  Persistent CTAs (one per SM, 512 TMEM columns = two
// accumulators), warp roles:
//   warps 0 .. TC_EPW-1  epilogue: TMEM -> registers -> bytesum_reduce -> coalesced stores (warp w:
//              lanes 32 (w % 4) .. +31, targets t = w / 4 (mod TC_EPW / 4), four targets in flight)
//   next 4 warps producers: cp.async of the next tiles' input words into TC_SA shared stages; their
//              first thread issues the tcgen05.mma of a tile (K / 32 instructions) and commits.
#ifndef HKS_TC_SA
#define HKS_TC_SA 2
#endif
#ifndef HKS_TC_MAXREG
#define HKS_TC_MAXREG 0
#endif
#ifndef HKS_TC_EPW
#define HKS_TC_EPW 16
#endif
#define TC_SA HKS_TC_SA
#define TC_EPW HKS_TC_EPW                  // epilogue warps (multiple of 4)
#define TC_THREADS ((TC_EPW + 4) * 32)

#ifdef BC_TRACE
__device__ long long g_bc_trace[6 * 64];   // events 0-4 per tile; event 5: kernel entry, after prologue, after griddepcontrol.wait
extern "C" void *hks_debug_bc_trace() {
    void *p = nullptr;
    cudaGetSymbolAddress(&p, g_bc_trace);
    return p;
}
#define BC_T(ev, j) do { if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64) g_bc_trace[(ev) * 64 + (j)] = clock64(); } while (0)
#else
#define BC_T(ev, j) do { } while (0)
#endif
template <int NSRC, bool LAZY>
#if HKS_TC_MAXREG   // a register cap below the full register file: room for other kernels' CTAs on the SM
__global__ void __maxnreg__(HKS_TC_MAXREG) k_bconv_tc(const __grid_constant__ BconvArgs A) {
#else
__global__ void __launch_bounds__(TC_THREADS, 1) k_bconv_tc(const __grid_constant__ BconvArgs A) {
#endif
    pdl_trigger();
    if (threadIdx.x == 0) BC_T(5, 0);
    constexpr int KPAD = 32 * ((NSRC + 3) / 4);   // bytes of K (whole K = 32 MMA steps)
    constexpr int NCH = KPAD / 16;                // 16-byte K chunks
    constexpr u32 SBO = NCH * 128;                // 8-row group stride
    constexpr u32 ATILE = 128 * KPAD;             // bytes per input stage
    const BconvGroup &G = A.g[blockIdx.y];
    const u32 tch = A.cw;                         // targets per z-chunk (even, <= 32)
    const u32 u0 = blockIdx.z * tch;
    if (u0 >= G.ndst) return;
    const u32 nt = min(tch, G.ndst - u0);
    const u32 ncol = 8 * ((nt + 1) & ~1u);        // MMA N (multiple of 16, <= 256)
    const size_t N = (size_t)1 << A.log_n;
    const u32 ntiles_all = (u32)(N >> 7);
    const u32 ntile = blockIdx.x < ntiles_all ? (ntiles_all - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    extern __shared__ __align__(1024) uint8_t tsm[];
    uint8_t *sB = tsm;                                   // 256 x KPAD
    uint8_t *sA = tsm + 256 * KPAD;                      // TC_SA x ATILE
    __shared__ __align__(8) u64 bar_done[2], bar_empty[2], bar_free[TC_SA];
    __shared__ u32 tmem_base_s;
    __shared__ ulonglong2 sred[32];                // per target: (2^64 - p, floor(2^80 / p))
    __shared__ u64 *sdst[32];                       // per target: output limb
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- prologue (before griddepcontrol.wait: ctx tables only) ----
    // B operand: the group's precomputed image (nt targets x SBO bytes, contiguous) by one bulk copy on its own
    // mbarrier (awaited by the MMA issuer only), plus zero rows for the padding target of an odd nt
    __shared__ __align__(8) u64 bar_img;
    {
        const u32 nimg = nt * (SBO / 16), ntot = (ncol / 8) * (SBO / 16);
        if (tid == 0) {
            mbar_init(smem_u32(&bar_img), 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_img)), "r"(nimg * 16)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(sB)),
                         "l"(G.mimg + (size_t)bconv_img_words(NSRC) * u0), "r"(nimg * 16), "r"(smem_u32(&bar_img))
                         : "memory");
        }
        for (u32 idx = nimg + tid; idx < ntot; idx += TC_THREADS) reinterpret_cast<uint4 *>(sB)[idx] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(smem_u32(&bar_done[b]), 1);
            mbar_init(smem_u32(&bar_empty[b]), TC_EPW);
        }
        for (int s = 0; s < TC_SA; s++) mbar_init(smem_u32(&bar_free[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // sB visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const u32 tmem = tmem_base_s;
    if (threadIdx.x == 0) BC_T(5, 1);
    pdl_wait();
    if (threadIdx.x == 0) BC_T(5, 2);

    if (warp >= TC_EPW) {
        // ---------------- producers + MMA issuer ----------------
        const u32 ptid = tid - TC_EPW * 32;       // 0..127: coefficient row m of the tile
        const u32 m = ptid;
        const u32 soff = (m >> 3) * SBO + (m & 7) * 16;
        const u64 *srcp[NSRC];
#pragma unroll
        for (int i = 0; i < NSRC; i++) srcp[i] = bc_src(A, G, i, N) + m;
        auto load_tile = [&](u32 j) {
            const u32 st = j % TC_SA;
            const size_t x0 = (size_t)(blockIdx.x + j * gridDim.x) << 7;
            const u32 base = smem_u32(sA + st * ATILE) + soff;
#pragma unroll
            for (int i = 0; i < NSRC; i++) cp_async8(base + (i >> 1) * 128 + (i & 1) * 8, srcp[i] + x0);
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        const u32 idesc = (2u << 4) | ((ncol >> 3) << 17) | ((128u >> 4) << 24);   // s32 += u8 x u8, K-major
        for (u32 j = 0; j + 1 < TC_SA; j++) {   // TC_SA - 1 groups in flight (empty ones past the end)
            if (j < ntile) load_tile(j);
            else asm volatile("cp.async.commit_group;" ::: "memory");
        }
        for (u32 j = 0; j < ntile; j++) {
            const u32 jn = j + TC_SA - 1;
            if (jn < ntile) {
                if (jn >= TC_SA) mbar_wait(smem_u32(&bar_free[jn % TC_SA]), (jn / TC_SA - 1) & 1);
                load_tile(jn);
            } else {
                asm volatile("cp.async.commit_group;" ::: "memory");   // keep the group count uniform
            }
            if (ptid == 0) BC_T(0, j);
            asm volatile("cp.async.wait_group %0;" ::"n"(TC_SA - 1) : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (ptid == 0) BC_T(1, j);
            if (ptid == 0) {
                const u32 b = j & 1;
                if (j == 0) mbar_wait(smem_u32(&bar_img), 0);
                if (j >= 2) mbar_wait(smem_u32(&bar_empty[b]), ((j >> 1) - 1) & 1);
                tc_fence_after();
                const u32 abase = smem_u32(sA + (j % TC_SA) * ATILE), bbase = smem_u32(sB);
#pragma unroll
                for (int s = 0; s < KPAD / 32; s++)
                    tc_mma_i8(tmem + b * 256, tc_desc(abase + s * 256, 128, SBO), tc_desc(bbase + s * 256, 128, SBO),
                              idesc, s > 0 ? 1u : 0u);
                tc_commit(smem_u32(&bar_free[j % TC_SA]));
                tc_commit(smem_u32(&bar_done[b]));
                BC_T(2, j);
            }
        }
    } else {
        // ---------------- epilogue ----------------
        // warp (quarter q, h) reduces a contiguous run of up to 8 targets: two 32-column TMEM loads and one
        // wait per tile (the accumulator is released before the reductions), so that eight independent
        // reductions are in flight per thread
        constexpr u32 NH = TC_EPW / 4;           // warps sharing a TMEM lane quarter
        constexpr u32 NCH = ((32 + NH - 1) / NH + 7) / 8;   // 8-target chunks of a run (1 at 16 epilogue warps)
        const u32 q = warp & 3, h = warp >> 2;
        const u32 lrow = q * 32 + lane;           // TMEM lane = coefficient row of the tile
        const u32 tpw = (nt + NH - 1) / NH;       // <= 8 NCH (nt <= 32)
        const u32 tb0 = h * tpw, tcnt = nt > tb0 ? min(tpw, nt - tb0) : 0;
        // per-target reduction constants and output limbs of this run, written by the run's quarter-0 warp and
        // shared with the other three lane quarters through a named barrier (ids 2 + h): the global loads
        // stay off the CTA-wide prologue barrier
        if (q == 0 && (u32)lane < tcnt) {
            const u32 t = tb0 + lane;
            const PrimeConst pc = A.pc[G.dst_prime[u0 + t]];
            sred[t] = make_ulonglong2(0 - pc.p, pc.mu80);
            sdst[t] = A.out + (size_t)G.dst_slot[u0 + t] * N;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory");
        for (u32 j = 0; j < ntile; j++) {
            const u32 b = j & 1;
            mbar_wait(smem_u32(&bar_done[b]), (j >> 1) & 1);
            if (warp == 0 && lane == 0) BC_T(3, j);
            tc_fence_after();
            const size_t x = ((size_t)(blockIdx.x + j * gridDim.x) << 7) + lrow;
            if (NCH == 1) {
            const u32 tbase = tmem + b * 256 + ((q * 32) << 16) + tb0 * 8;
            u32 v[2][32];
            if (tcnt > 0) tc_ld32(tbase, v[0]);
            if (tcnt > 4) tc_ld32(tbase + 32, v[1]);
            tc_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_empty[b]));
            // branch-free over the eight slots (a slot past the run reduces target tb0 again and is not stored),
            // so that the eight reductions interleave instead of running one predicated block after another
#pragma unroll
            for (int hh = 0; hh < 2; hh++) {
                u64 o[4];
                u64 *dp[4];
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    const u32 k = 4 * hh + kk;
                    const u32 t = tb0 + (k < tcnt ? k : 0u);
                    const ulonglong2 c = sred[t];
                    const u32 *r = &v[hh][8 * kk];
                    o[kk] = bytesum_reduce_c<LAZY>(r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], c.x, (u32)c.y);
                    dp[kk] = sdst[t] + x;
                }
#pragma unroll
                for (int kk = 0; kk < 4; kk++)
                    if ((u32)(4 * hh + kk) < tcnt) *dp[kk] = o[kk];
            }
            } else {   // fewer epilogue warps (HKS_TC_EPW < 16): the run is reduced in chunks of eight targets
#pragma unroll 1
            for (u32 ch = 0; ch < NCH; ch++) {
                const u32 cb = tb0 + 8 * ch;   // first target of this chunk
                const u32 ccnt = tcnt > 8 * ch ? min(8u, tcnt - 8 * ch) : 0u;
                const u32 tbase = tmem + b * 256 + ((q * 32) << 16) + cb * 8;
                u32 v[2][32];
                if (ccnt > 0) tc_ld32(tbase, v[0]);
                if (ccnt > 4) tc_ld32(tbase + 32, v[1]);
                tc_wait_ld();
                if (ch == NCH - 1) {   // the accumulator is released once its last chunk is in registers
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&bar_empty[b]));
                }
                // branch-free over the eight slots (a slot past the run reduces target cb again and is not
                // stored), so that the eight reductions interleave instead of running one predicated block after
                // another
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    u64 o[4];
                    u64 *dp[4];
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) {
                        const u32 k = 4 * hh + kk;
                        const u32 t = min(cb + (k < ccnt ? k : 0u), 31u);
                        const ulonglong2 c = sred[t];
                        const u32 *r = &v[hh][8 * kk];
                        o[kk] = bytesum_reduce_c<LAZY>(r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], c.x, (u32)c.y);
                        dp[kk] = sdst[t] + x;
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                        if ((u32)(4 * hh + kk) < ccnt) *dp[kk] = o[kk];
                }
            }
            }
            if (warp == 0 && lane == 0) BC_T(4, j);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int NSRC>
static hks_status bconv_tc_go(const BconvArgs &a, cudaStream_t s) {
    constexpr int KPAD = 32 * ((NSRC + 3) / 4);
    const size_t smem = 256 * KPAD + TC_SA * 128 * KPAD;
    const int nsm = hks_num_sms();
    hks_func_smem((const void *)k_bconv_tc<NSRC, true>, smem);
    hks_func_smem((const void *)k_bconv_tc<NSRC, false>, smem);
    const size_t N = (size_t)1 << a.log_n;
    u32 maxdst = 0;
    for (u32 g = 0; g < a.ngroups; g++) maxdst = max(maxdst, a.g[g].ndst);
    const u32 nz = (maxdst + 31) / 32;
    u32 tch = (maxdst + nz - 1) / nz;
    tch = (tch + 1) & ~1u;
    BconvArgs b = a;
    b.cw = tch;
    // one CTA per SM (512 TMEM columns each): split the SMs over (group, target chunk) pairs
    const u32 pairs = a.ngroups * nz;
    u32 gx = std::max<u32>(1, (u32)nsm / pairs);
    gx = std::min<u32>(gx, (u32)(N >> 7));
    ProfScope ps(K_BCONV, s);
    cudaError_t e;
    const bool pdl = pdl_enabled() && !a.fresh_tables;
    if (a.lazy_out)
        e = hks_launch_pdl(pdl, k_bconv_tc<NSRC, true>, dim3(gx, a.ngroups, nz), dim3(TC_THREADS), smem, s, b);
    else
        e = hks_launch_pdl(pdl, k_bconv_tc<NSRC, false>, dim3(gx, a.ngroups, nz), dim3(TC_THREADS), smem, s, b);
    double words = 0, macs = 0;
    for (u32 g = 0; g < a.ngroups; g++) {
        words += a.g[g].nsrc + a.g[g].ndst;
        macs += (double)a.g[g].nsrc * a.g[g].ndst;
    }
    (void)macs;   // the contraction runs on the tensor pipe (tcgen05): no integer-pipe products to count
    ps.done(words * (double)N * 8.0, 0.0);
    if (e != cudaSuccess) HKS_FAIL(HKS_ECUDA, "k_bconv_tc launch: %s", cudaGetErrorString(e));
    return HKS_OK;
}

// enough 128-coefficient tiles to give every SM one (otherwise the tensor kernels' fixed prologue loses)
bool bconv_tc_large(u32 log_n, u32 ngroups) {
    const int nsm = hks_num_sms();
    return (((size_t)1 << log_n) >> 7) * ngroups >= (size_t)nsm;
}

struct ScaleArgs {
    const u64 *in;
    u64 *out;
    const u64 *w;          // device: w[0..nl), then the Shoup companions
    u64 p[BC_MAXSRC];
    u32 nl, log_n;
};
__global__ void __launch_bounds__(256) k_limb_scale(const __grid_constant__ ScaleArgs A) {
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << A.log_n;
    const u32 i = blockIdx.y;
    const size_t x = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (x >= N) return;
    const u64 w = A.w[i], wp = A.w[A.nl + i];
    const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(A.in + i * N + x);
    *reinterpret_cast<ulonglong2 *>(A.out + i * N + x) = make_ulonglong2(shoup(v.x, w, wp, A.p[i]), shoup(v.y, w, wp, A.p[i]));
}

hks_status launch_limb_scale(const u64 *in, u64 *out, u32 nl, const u64 *dw, const u64 *p, u32 log_n, cudaStream_t s) {
    if (nl < 1 || nl > BC_MAXSRC) HKS_FAIL(HKS_EINVAL, "limb_scale: %u limbs", nl);
    ScaleArgs a{};
    a.in = in;
    a.out = out;
    a.w = dw;
    a.nl = nl;
    a.log_n = log_n;
    for (u32 i = 0; i < nl; i++) a.p[i] = p[i];
    const size_t N = (size_t)1 << log_n;
    (void)hks_launch(k_limb_scale, dim3((u32)(N / 2 / 256), nl), dim3(256), 0, s, a);
    HKS_CHECK_LAUNCH();
    return HKS_OK;
}

// hks_evk_prepare: key limb t < nq (the Q limbs of every digit and both components) times [P^-1]_{q_t}
// (canonical Shoup product), the P limbs copied; elementwise, so in place is allowed.
struct EvkPrepArgs {
    const u64 *in;
    u64 *out;
    const ulonglong2 *pinv;    // [nq] (P^-1 mod q_t, Shoup companion)
    const PrimeConst *pc;
    u32 nq, nk, log_n;
};
__global__ void __launch_bounds__(256) k_evk_prepare(const __grid_constant__ EvkPrepArgs A) {
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << A.log_n;
    const u32 limb = blockIdx.y, t = limb % A.nk;
    const size_t x = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (x >= N) return;
    const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(A.in + limb * N + x);
    ulonglong2 r = v;
    if (t < A.nq) {
        const ulonglong2 w = A.pinv[t];
        const u64 p = A.pc[t].p;
        r = make_ulonglong2(shoup(v.x, w.x, w.y, p), shoup(v.y, w.x, w.y, p));
    }
    *reinterpret_cast<ulonglong2 *>(A.out + limb * N + x) = r;
}

hks_status launch_evk_prepare(const hks_ctx *c, const u64 *in, u64 *out, u32 ndig, cudaStream_t s) {
    EvkPrepArgs a{};
    a.in = in;
    a.out = out;
    a.pinv = c->d_pinv;
    a.pc = c->d_pc;
    a.nq = c->nq;
    a.nk = c->nq + c->np;
    a.log_n = c->log_n;
    const size_t N = (size_t)1 << c->log_n;
    const u32 bx = (u32)std::max<size_t>(1, N / 2 / 256);
    (void)hks_launch(k_evk_prepare, dim3(bx, 2 * ndig * a.nk), dim3(256), 0, s, a);
    HKS_CHECK_LAUNCH();
    return HKS_OK;
}

// hks_bconv's constants for an arbitrary (src, dst) prime pair (Eq. 1, §3.6.3), built on
// the device so that the generic entry point needs no host->device copy (graph-capturable):
//   thread (i, u), i < 4 ceil(nsrc / 4):  v = [qhat_i]_{t_u} = prod_{k != i} q_k mod t_u -> mat (30-bit
//       halves) and the 8 byte-column words of v (word c holds byte c of 2^(8a) v mod t in byte a) placed
//       in the k_bconv_tc B image (zero rows for i >= nsrc);
//   thread i < nsrc:  w_i = [qhat_i^-1]_{q_i} = h^(q_i - 2), h = prod_{k != i} q_k mod q_i, and
//       floor(w_i 2^64 / q_i).
// Host-only work stays with the caller: the primes travel in the parameter block.
struct BconvPrepArgs {
    u64 src[BC_MAXSRC];
    u64 dst[2 * BC_MAXDST];
    u32 nsrc, ndst;
    u64 *w;
    uint2 *mat;
    u64 *img;
};
__device__ __forceinline__ u64 prep_mulmod(u64 a, u64 b, u64 m) {
    return (u64)((unsigned __int128)a * b % m);
}
__global__ void __launch_bounds__(256) k_bconv_prep(const __grid_constant__ BconvPrepArgs A) {
    pdl_trigger();
    pdl_wait();   // the workspace may still be read by the previous call's conversion
    const u32 nrow = 4 * ((A.nsrc + 3) / 4);
    const u32 nent = nrow * A.ndst;
    const u32 iw = bconv_img_words(A.nsrc);
    for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < nent + A.nsrc; e += gridDim.x * blockDim.x) {
        if (e < nent) {
            const u32 i = e / A.ndst, u = e - i * A.ndst;
            const u64 t = A.dst[u];
            u64 v = 0;
            if (i < A.nsrc) {
                v = 1;
                for (u32 k = 0; k < A.nsrc; k++)
                    if (k != i) v = prep_mulmod(v, A.src[k] % t, t);
                A.mat[(size_t)i * A.ndst + u] = make_uint2((u32)(v & 0x3fffffffu), (u32)(v >> 30));
            }
            u64 m[8];
            m[0] = v;
            for (int a = 1; a < 8; a++) m[a] = prep_mulmod(m[a - 1], 256, t);
            // image word (u, kc, c, h) with source i = 2 kc + h
            u64 *dst = A.img + (size_t)u * iw + (size_t)(i >> 1) * 16 + (i & 1);
            for (int c = 0; c < 8; c++) {
                u64 wd = 0;
                for (int a = 0; a < 8; a++) wd |= ((m[a] >> (8 * c)) & 0xffull) << (8 * a);
                dst[2 * c] = wd;
            }
        } else {
            const u32 i = e - nent;
            const u64 q = A.src[i];
            u64 h = 1;
            for (u32 k = 0; k < A.nsrc; k++)
                if (k != i) h = prep_mulmod(h, A.src[k] % q, q);
            u64 w = 1, b = h;
            for (u64 ex = q - 2; ex; ex >>= 1, b = prep_mulmod(b, b, q))
                if (ex & 1) w = prep_mulmod(w, b, q);
            A.w[i] = w;
            A.w[A.nsrc + i] = (u64)(((unsigned __int128)w << 64) / q);
        }
    }
}

hks_status launch_bconv_prep(const u64 *src, u32 nsrc, const u64 *dst, u32 ndst, u64 *w, uint2 *mat, u64 *img,
                             cudaStream_t s) {
    if (nsrc < 1 || nsrc > BC_MAXSRC || ndst < 1 || ndst > 2 * BC_MAXDST) HKS_FAIL(HKS_EINVAL, "bconv_prep: sizes");
    BconvPrepArgs a{};
    for (u32 i = 0; i < nsrc; i++) a.src[i] = src[i];
    for (u32 u = 0; u < ndst; u++) a.dst[u] = dst[u];
    a.nsrc = nsrc;
    a.ndst = ndst;
    a.w = w;
    a.mat = mat;
    a.img = img;
    const u32 n = 4 * ((nsrc + 3) / 4) * ndst + nsrc;
    (void)hks_launch(k_bconv_prep, dim3((n + 255) / 256), dim3(256), 0, s, a);
    HKS_CHECK_LAUNCH();
    return HKS_OK;
}

#if HKS_EXPERIMENTAL
// Experimental build only (-DHKS_EXPERIMENTAL=1, tools/build_variant.sh): HKS_BCONV_TC=0 selects the
// warp-level IMMA kernel, HKS_BCONV_MMA=0 the integer-pipe kernels, HKS_BCONV_KARA=0 the plain integer
// kernel, HKS_BCONV_FP=1 the FP64-assisted one (slower: 60 vs 52 us for the C2 ModUp conversion, the
// 128-bit recombination of the FP64 limb sums makes it issue-bound), HKS_NTT_TC=1 the tensor-core NTT
// column pass (results identical; tests/test_gpu_parity.py::test_bconv_alternate_paths_identical).  The
// product library has one path per op and reads no environment switch.
static bool env_flag(const char *name, bool dflt) {
    const char *e = getenv(name);
    return e ? e[0] == '1' : dflt;
}
static bool getenv_tc_enabled() { static const bool on = env_flag("HKS_BCONV_TC", true); return on; }
static bool getenv_mma_enabled() { static const bool on = env_flag("HKS_BCONV_MMA", true); return on; }
static bool getenv_kara_enabled() { static const bool on = env_flag("HKS_BCONV_KARA", true); return on; }
static bool getenv_fp_enabled() { static const bool on = env_flag("HKS_BCONV_FP", false); return on; }
bool ntt_tc_enabled() { static const bool on = env_flag("HKS_NTT_TC", HKS_NTT_TC_DEFAULT != 0); return on; }
#else
static bool getenv_tc_enabled() { return true; }
static bool getenv_mma_enabled() { return true; }
static bool getenv_kara_enabled() { return true; }
bool ntt_tc_enabled() { return HKS_NTT_TC_DEFAULT != 0; }
#endif
bool bconv_tc_enabled() { return getenv_mma_enabled() && getenv_tc_enabled(); }

#if HKS_EXPERIMENTAL
// FP64-assisted variant (B200: the FP64 pipe runs 64 DFMA/clk/SM and is otherwise idle here):
// sources [0, NSRC - NFP) accumulate on the integer pipe (4 IMAD.WIDE per MAC), sources
// [NSRC - NFP, NSRC) on the FP64 pipe (9 exact DFMA per MAC on 20-bit limbs), one coefficient per
// thread; both partial sums are added as 128-bit integers before the single reduction.  The result
// is the same integer X = sum_i y_i [qhat_i]_t, so the output is bit-identical to k_bconv.
template <int NSRC, int NFP, bool LAZY>
__global__ void __launch_bounds__(256) k_bconv_fp(const __grid_constant__ BconvArgs A) {
    pdl_trigger();
    constexpr int NINT = NSRC - NFP;
    const BconvGroup &G = A.g[blockIdx.y];
    const u32 u0 = blockIdx.z * BC_TCH;
    if (u0 >= G.ndst) return;
    const u32 nt = min((u32)BC_TCH, G.ndst - u0);
    __shared__ uint2 smat[(NINT > 0 ? NINT : 1) * BC_TCH];
    __shared__ double smatf[NFP * BC_TCH * 3];
    __shared__ PrimeConst spc[BC_TCH];
    for (u32 idx = threadIdx.x; idx < NSRC * nt; idx += blockDim.x) {
        const u32 i = idx / nt, u = idx - i * nt;
        if ((int)i < NINT) {
            smat[i * BC_TCH + u] = G.mat[(size_t)i * G.mat_stride + u0 + u];
        } else {
            const double *f = G.matf + ((size_t)i * G.mat_stride + u0 + u) * 3;
            double *d = smatf + ((i - NINT) * BC_TCH + u) * 3;
            d[0] = f[0];
            d[1] = f[1];
            d[2] = f[2];
        }
    }
    for (u32 u = threadIdx.x; u < nt; u += blockDim.x) spc[u] = A.pc[G.dst_prime[u0 + u]];
    __syncthreads();
    pdl_wait();   // ctx tables above are immutable; the inputs below come from the predecessor

    const size_t N = (size_t)1 << A.log_n;
    const size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= N) return;
    u32 yl[NINT > 0 ? NINT : 1], yh[NINT > 0 ? NINT : 1];
    double Y[NFP][3];
#pragma unroll
    for (int i = 0; i < NSRC; i++) {
        const u64 v = bc_src(A, G, i, N)[x];
        if (i < NINT)
            split30(v, yl[i], yh[i]);
        else
            split20d(v, Y[i - NINT][0], Y[i - NINT][1], Y[i - NINT][2]);
    }
    for (u32 u = 0; u < nt; u++) {
        Acc30 a;
        if (NINT > 0) {
            const uint2 m = smat[u];
            acc_first(a, yl[0], yh[0], m.x, m.y);
#pragma unroll
            for (int i = 1; i < NINT; i++) {
                const uint2 mm = smat[i * BC_TCH + u];
                acc_mac(a, yl[i], yh[i], mm.x, mm.y);
            }
        }
        AccF f;
        {
            const double *m = smatf + u * 3;
            accf_first(f, Y[0][0], Y[0][1], Y[0][2], m[0], m[1], m[2]);
        }
#pragma unroll
        for (int i = 1; i < NFP; i++) {
            const double *m = smatf + (i * BC_TCH + u) * 3;
            accf_mac(f, Y[i][0], Y[i][1], Y[i][2], m[0], m[1], m[2]);
        }
        u64 lo = 0, hi = 0;
        if (NINT > 0) acc_to128(a, lo, hi);
        accf_add128(f, lo, hi);
        const PrimeConst pc = spc[u];
        A.out[(size_t)G.dst_slot[u0 + u] * N + x] = LAZY ? reduce128_lazy(lo, hi, pc) : reduce128(lo, hi, pc);
    }
}

template <int NSRC, int NFP>
static void bconv_fp_go(const BconvArgs &a, cudaStream_t s) {
    const u32 threads = 256;
    const size_t N = (size_t)1 << a.log_n;
    u32 maxdst = 0;
    for (u32 g = 0; g < a.ngroups; g++) maxdst = max(maxdst, a.g[g].ndst);
    dim3 grid((u32)((N + threads - 1) / threads), a.ngroups, (maxdst + BC_TCH - 1) / BC_TCH);
    ProfScope ps(K_BCONV, s);
    if (a.lazy_out)
        (void)hks_launch(k_bconv_fp<NSRC, NFP, true>, grid, dim3(threads), 0, s, a);
    else
        (void)hks_launch(k_bconv_fp<NSRC, NFP, false>, grid, dim3(threads), 0, s, a);
    double words = 0, macs = 0;
    for (u32 g = 0; g < a.ngroups; g++) {
        words += a.g[g].nsrc + a.g[g].ndst;
        macs += (double)a.g[g].nsrc * a.g[g].ndst;
    }
    ps.done(words * (double)N * 8.0, macs * (double)N * 4.0);
}

#endif  // HKS_EXPERIMENTAL

#ifndef HKS_BCONV_CPT
#define HKS_BCONV_CPT 1
#endif
template <int NSRC>
static void bconv_go(const BconvArgs &a, cudaStream_t s) {
    constexpr int CPT = HKS_BCONV_CPT;   // coefficients per thread
    const u32 threads = 256;
    const size_t N = (size_t)1 << a.log_n;
    u32 maxdst = 0;
    for (u32 g = 0; g < a.ngroups; g++) maxdst = max(maxdst, a.g[g].ndst);
    dim3 grid((u32)((N / CPT + threads - 1) / threads), a.ngroups, (maxdst + BC_TCH - 1) / BC_TCH);
    ProfScope ps(K_BCONV, s);
    if (a.lazy_out)
        (void)hks_launch(k_bconv<NSRC, true, CPT>, grid, dim3(threads), 0, s, a);
    else
        (void)hks_launch(k_bconv<NSRC, false, CPT>, grid, dim3(threads), 0, s, a);
    double words = 0, macs = 0;
    for (u32 g = 0; g < a.ngroups; g++) {
        words += a.g[g].nsrc + a.g[g].ndst;
        macs += (double)a.g[g].nsrc * a.g[g].ndst;
    }
    ps.done(words * (double)N * 8.0, macs * (double)N * 4.0);
}

hks_status launch_bconv(const BconvArgs &a, u32 /*max_ndst*/, cudaStream_t s) {
    // all groups of one launch share nsrc (the caller groups them so)
#if HKS_EXPERIMENTAL
    if (a.g[0].matf && getenv_fp_enabled()) {
        // FP64-pipe share chosen so both pipes carry similar work: 16 NINT + 56 ~ 18 NFP + 10 cycles
        switch (a.g[0].nsrc) {
            case 6: bconv_fp_go<6, 3>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 7: bconv_fp_go<7, 4>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 8: bconv_fp_go<8, 4>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 9: bconv_fp_go<9, 5>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 10: bconv_fp_go<10, 6>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 11: bconv_fp_go<11, 6>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 12: bconv_fp_go<12, 7>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 13: bconv_fp_go<13, 7>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 14: bconv_fp_go<14, 8>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 15: bconv_fp_go<15, 8>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            case 16: bconv_fp_go<16, 9>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            default: break;
        }
    }
#endif
    // the tensor-core kernels pay a fixed prologue (TMEM allocation, matrix image, barriers): small
    // conversions (fewer 128-coefficient tiles than SMs, e.g. N = 2^12) stay on the integer pipe
    const bool large = bconv_tc_large(a.log_n, a.ngroups);
    if (a.big && large && a.g[0].mimg && getenv_mma_enabled() && getenv_tc_enabled()) {
        switch (a.g[0].nsrc) {
#define CT(NS) case NS: return bconv_tc_go<NS>(a, s);
            CT(1) CT(2) CT(3) CT(4) CT(5) CT(6) CT(7) CT(8) CT(9) CT(10) CT(11) CT(12) CT(13) CT(14) CT(15) CT(16)
#undef CT
            default: break;
        }
    }
#if HKS_EXPERIMENTAL
    if (a.big && large && a.g[0].matb && getenv_mma_enabled() && !getenv_tc_enabled()) {
        switch (a.g[0].nsrc) {
#define CM(NS) case NS: bconv_mma_go<NS>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            CM(1) CM(2) CM(3) CM(4) CM(5) CM(6) CM(7) CM(8) CM(9) CM(10) CM(11) CM(12) CM(13) CM(14) CM(15) CM(16)
#undef CM
            default: break;
        }
    }
#endif
    if (a.g[0].mats && getenv_kara_enabled()) {
        switch (a.g[0].nsrc) {
#define CK(NS) case NS: bconv_kara_go<NS>(a, s); HKS_CHECK_LAUNCH(); return HKS_OK;
            CK(2) CK(3) CK(4) CK(5) CK(6) CK(7) CK(8) CK(9) CK(10) CK(11)   // 12: spills at 3 CTAs / SM
#undef CK
            default: break;
        }
    }
    switch (a.g[0].nsrc) {
#define C(NS) case NS: bconv_go<NS>(a, s); break;
        C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10) C(11) C(12) C(13) C(14) C(15) C(16)
#undef C
        default:
            HKS_FAIL(HKS_EINVAL, "bconv: nsrc %u out of range", a.g[0].nsrc);
    }
    HKS_CHECK_LAUNCH();
    return HKS_OK;
}

// ------------------------------------------------------------------------------------------------
// Key inner product (§3.6.5 dot-product fusion):
//   acc0[t] = sum_j D_j[t] * b_j[t],  acc1[t] = sum_j D_j[t] * a_j[t]   (mod t)
// with D_j optionally read through the EVAL automorphism (hoisted rotation, reading 14).
// grid.x: coefficient blocks, grid.y: extended limb t.
// any digit count (runtime loop, 30-bit-split MACs: up to 16 digits)
__global__ void __launch_bounds__(256) k_kip_any(const __grid_constant__ KipArgs A) {
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << A.log_n;
    const u32 t = blockIdx.y;
    const size_t x0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (x0 >= N) return;
    const u32 prime = t <= A.level ? t : A.nq + (t - A.level - 1);   // key limb index == prime index
    const PrimeConst pc = A.pc[prime];
    Acc30 a0[2], a1[2];
    acc_zero(a0[0]); acc_zero(a0[1]);
    acc_zero(a1[0]); acc_zero(a1[1]);
    u32 s0 = 0, s1 = 1;
    if (A.galois != 1) {
        s0 = automorph_src((u32)x0, A.log_n, A.galois);
        s1 = automorph_src((u32)x0 + 1, A.log_n, A.galois);
    }
    for (u32 j = 0; j < A.beta; j++) {
        const bool own = A.c1 && t <= A.level && t / A.alpha == j;
        const u64 *D = own ? A.c1 + (size_t)t * N : A.ext + ((size_t)j * A.ne + t) * N;
        u64 d0, d1;
        if (A.galois == 1) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(D + x0);
            d0 = v.x;
            d1 = v.y;
        } else {
            d0 = D[s0];
            d1 = D[s1];
        }
        const ulonglong2 kb = *reinterpret_cast<const ulonglong2 *>(A.evk + (((size_t)j * 2 + 0) * A.nk + prime) * N + x0);
        const ulonglong2 ka = *reinterpret_cast<const ulonglong2 *>(A.evk + (((size_t)j * 2 + 1) * A.nk + prime) * N + x0);
        u32 dl, dh, ml, mh;
        split30(d0, dl, dh);
        split30(kb.x, ml, mh); acc_mac(a0[0], dl, dh, ml, mh);
        split30(ka.x, ml, mh); acc_mac(a1[0], dl, dh, ml, mh);
        split30(d1, dl, dh);
        split30(kb.y, ml, mh); acc_mac(a0[1], dl, dh, ml, mh);
        split30(ka.y, ml, mh); acc_mac(a1[1], dl, dh, ml, mh);
    }
    ulonglong2 o0, o1;
    o0.x = acc_reduce(a0[0], pc);
    o0.y = acc_reduce(a0[1], pc);
    o1.x = acc_reduce(a1[0], pc);
    o1.y = acc_reduce(a1[1], pc);
    *reinterpret_cast<ulonglong2 *>(A.acc + (size_t)t * N + x0) = o0;
    *reinterpret_cast<ulonglong2 *>(A.acc + ((size_t)A.ne + t) * N + x0) = o1;
}

template <int BETA>
__global__ void __launch_bounds__(256) k_kip(const __grid_constant__ KipArgs A) {
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << A.log_n;
    const u32 t = blockIdx.y;
    const size_t x0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (x0 >= N) return;
    const u32 prime = t <= A.level ? t : A.nq + (t - A.level - 1);   // key limb index == prime index
    const u32 jown = (A.c1 && t <= A.level) ? t / A.alpha : 0xffffffffu;
    u32 s0 = 0, s1 = 1;
    if (A.galois != 1) {
        s0 = automorph_src((u32)x0, A.log_n, A.galois);
        s1 = automorph_src((u32)x0 + 1, A.log_n, A.galois);
    }
    ulonglong2 kb[BETA], ka[BETA];
    u64 d0[BETA], d1[BETA];
#pragma unroll
    for (int j = 0; j < BETA; j++) {
        const u64 *D = (u32)j == jown ? A.c1 + (size_t)t * N : A.ext + ((size_t)j * A.ne + t) * N;
        if (A.galois == 1) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(D + x0);
            d0[j] = v.x;
            d1[j] = v.y;
        } else {
            d0[j] = D[s0];
            d1[j] = D[s1];
        }
        kb[j] = *reinterpret_cast<const ulonglong2 *>(A.evk + (((size_t)j * 2 + 0) * A.nk + prime) * N + x0);
        ka[j] = *reinterpret_cast<const ulonglong2 *>(A.evk + (((size_t)j * 2 + 1) * A.nk + prime) * N + x0);
    }
    // Karatsuba products (3 IMAD.WIDE each); D split once per term, shared by the two key words
    AccK a0[2], a1[2];
#pragma unroll
    for (int j = 0; j < BETA; j++) {
        u32 dl, dh, ml, mh;
#define KKP(J)                                                                                    \
        if (j == J) {                                                                             \
            split30(d0[J], dl, dh);                                                               \
            u32 ds = dl + dh;                                                                     \
            split30(kb[J].x, ml, mh); acck_mac<J>(a0[0], dl, dh, ds, ml, mh, ml + mh);            \
            split30(ka[J].x, ml, mh); acck_mac<J>(a1[0], dl, dh, ds, ml, mh, ml + mh);            \
            split30(d1[J], dl, dh);                                                               \
            ds = dl + dh;                                                                         \
            split30(kb[J].y, ml, mh); acck_mac<J>(a0[1], dl, dh, ds, ml, mh, ml + mh);            \
            split30(ka[J].y, ml, mh); acck_mac<J>(a1[1], dl, dh, ds, ml, mh, ml + mh);            \
        }
        KKP(0) KKP(1) KKP(2) KKP(3)
#undef KKP
    }
    const PrimeConst pc = A.pc[prime];
    u64 lo, hi;
    ulonglong2 o0, o1;
    acck_to128(a0[0], BETA, lo, hi); o0.x = reduce128(lo, hi, pc);
    acck_to128(a0[1], BETA, lo, hi); o0.y = reduce128(lo, hi, pc);
    acck_to128(a1[0], BETA, lo, hi); o1.x = reduce128(lo, hi, pc);
    acck_to128(a1[1], BETA, lo, hi); o1.y = reduce128(lo, hi, pc);
    *reinterpret_cast<ulonglong2 *>(A.acc + (size_t)t * N + x0) = o0;
    *reinterpret_cast<ulonglong2 *>(A.acc + ((size_t)A.ne + t) * N + x0) = o1;
}

hks_status launch_kip(const KipArgs &a, cudaStream_t s) {
    const u32 threads = 256;
    const size_t N = (size_t)1 << a.log_n;
    dim3 grid((u32)((N / 2 + threads - 1) / threads), a.ne);
    ProfScope ps(K_KIP, s);
    switch (a.beta) {
        case 1: (void)hks_launch(k_kip<1>, grid, dim3(threads), 0, s, a); break;
        case 2: (void)hks_launch(k_kip<2>, grid, dim3(threads), 0, s, a); break;
        case 3: (void)hks_launch(k_kip<3>, grid, dim3(threads), 0, s, a); break;
        case 4: (void)hks_launch(k_kip<4>, grid, dim3(threads), 0, s, a); break;
        default: (void)hks_launch(k_kip_any, grid, dim3(threads), 0, s, a); break;
    }
    HKS_CHECK_LAUNCH();
    ps.done((3.0 * a.beta + 2.0) * a.ne * (double)N * 8.0,    // D_j + (b_j, a_j) read, acc0/acc1 written
            (double)a.ne * a.beta * 2.0 * (double)N * 4.0);
    return HKS_OK;
}

// Multi-ciphertext key inner product: the nct ciphertexts of a batch share one key, whose words are read
// from HBM once per batch (amortising the dominant key stream, SURVEY.md §7 "key streaming").
template <int BETA>
__global__ void __launch_bounds__(512) k_kip_multi(const __grid_constant__ KipMultiArgs A) {
    // one (ciphertext, coefficient block) per CTA; the nct CTAs sharing a key block are adjacent in
    // launch order (ciphertext fastest), so the key words come from HBM once and from L2 for the others.
    // Karatsuba products (3 IMAD.WIDE each), the digit count a template parameter (straight-line code).
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << A.log_n;
    const u32 t = blockIdx.y;
    const u32 xb = blockIdx.x / A.nct, c = blockIdx.x - xb * A.nct;
    const size_t x0 = ((size_t)xb * blockDim.x + threadIdx.x) * 2;
    if (x0 >= N) return;
    const u32 prime = t <= A.level ? t : A.nq + (t - A.level - 1);
    const u32 jown = (A.c1[c] && t <= A.level) ? t / A.alpha : 0xffffffffu;
    u32 s0 = (u32)x0, s1 = (u32)x0 + 1;
    if (A.galois != 1) {
        s0 = automorph_src((u32)x0, A.log_n, A.galois);
        s1 = automorph_src((u32)x0 + 1, A.log_n, A.galois);
    }
    ulonglong2 kb[BETA], ka[BETA];
    u64 d0[BETA], d1[BETA];
#pragma unroll
    for (int j = 0; j < BETA; j++) {
        kb[j] = *reinterpret_cast<const ulonglong2 *>(A.evk + (((size_t)j * 2 + 0) * A.nk + prime) * N + x0);
        ka[j] = *reinterpret_cast<const ulonglong2 *>(A.evk + (((size_t)j * 2 + 1) * A.nk + prime) * N + x0);
        const u64 *D = (u32)j == jown ? A.c1[c] + (size_t)t * N : A.ext[c] + ((size_t)j * A.ne + t) * N;
        d0[j] = D[s0];
        d1[j] = D[s1];
    }
    AccK a0[2], a1[2];
#pragma unroll
    for (int j = 0; j < BETA; j++) {
        u32 dl, dh, ml, mh;
#define KP(J, DV, KW, ACC)                                                                        \
        {                                                                                         \
            split30(KW, ml, mh);                                                                  \
            acck_mac<J>(ACC, dl, dh, ds, ml, mh, ml + mh);                                        \
        }
        split30(d0[j], dl, dh);
        u32 ds = dl + dh;
        if (j == 0) { KP(0, d0, kb[0].x, a0[0]) KP(0, d0, ka[0].x, a1[0]) }
        if (j == 1) { KP(1, d0, kb[1].x, a0[0]) KP(1, d0, ka[1].x, a1[0]) }
        if (j == 2) { KP(2, d0, kb[2].x, a0[0]) KP(2, d0, ka[2].x, a1[0]) }
        if (j == 3) { KP(3, d0, kb[3].x, a0[0]) KP(3, d0, ka[3].x, a1[0]) }
        split30(d1[j], dl, dh);
        ds = dl + dh;
        if (j == 0) { KP(0, d1, kb[0].y, a0[1]) KP(0, d1, ka[0].y, a1[1]) }
        if (j == 1) { KP(1, d1, kb[1].y, a0[1]) KP(1, d1, ka[1].y, a1[1]) }
        if (j == 2) { KP(2, d1, kb[2].y, a0[1]) KP(2, d1, ka[2].y, a1[1]) }
        if (j == 3) { KP(3, d1, kb[3].y, a0[1]) KP(3, d1, ka[3].y, a1[1]) }
#undef KP
    }
    const PrimeConst pc = A.pc[prime];
    u64 lo, hi;
    ulonglong2 o0, o1;
    acck_to128(a0[0], BETA, lo, hi); o0.x = reduce128(lo, hi, pc);
    acck_to128(a0[1], BETA, lo, hi); o0.y = reduce128(lo, hi, pc);
    acck_to128(a1[0], BETA, lo, hi); o1.x = reduce128(lo, hi, pc);
    acck_to128(a1[1], BETA, lo, hi); o1.y = reduce128(lo, hi, pc);
    *reinterpret_cast<ulonglong2 *>(A.acc[c] + (size_t)t * N + x0) = o0;
    *reinterpret_cast<ulonglong2 *>(A.acc[c] + ((size_t)A.ne + t) * N + x0) = o1;
}

hks_status launch_kip_multi(const KipMultiArgs &a, cudaStream_t s) {
    if (a.beta > 4 || a.nct > KIP_MAXCT) HKS_FAIL(HKS_EINVAL, "kip_multi: beta %u / nct %u", a.beta, a.nct);
#ifndef HKS_KIPM_THREADS
#define HKS_KIPM_THREADS 128   // measured: C3 7 649 (256) -> 7 720 rot-KS/s
#endif
    const u32 threads = HKS_KIPM_THREADS;
    const size_t N = (size_t)1 << a.log_n;
    dim3 grid((u32)((N / 2 + threads - 1) / threads) * a.nct, a.ne);
    ProfScope ps(K_KIP, s);
    switch (a.beta) {
        case 1: (void)hks_launch(k_kip_multi<1>, grid, dim3(threads), 0, s, a); break;
        case 2: (void)hks_launch(k_kip_multi<2>, grid, dim3(threads), 0, s, a); break;
        case 3: (void)hks_launch(k_kip_multi<3>, grid, dim3(threads), 0, s, a); break;
        default: (void)hks_launch(k_kip_multi<4>, grid, dim3(threads), 0, s, a); break;
    }
    HKS_CHECK_LAUNCH();
    ps.done((2.0 * a.beta + a.nct * (a.beta + 2.0)) * a.ne * (double)N * 8.0,
            (double)a.nct * a.ne * a.beta * 2.0 * (double)N * 4.0);
    return HKS_OK;
}

// ------------------------------------------------------------------------------------------------
// EVAL-form automorphism (SURVEY.md §8(c) reading 15): out[j] = in[j'].
// The permutation maps aligned 2^b blocks onto aligned 2^b blocks, so a warp's gather stays
// inside one 256-byte segment.
__global__ void __launch_bounds__(256) k_automorph(const u64 *__restrict__ in, u64 *__restrict__ out,
                                                  u32 log_n, u64 galois) {
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << log_n;
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t l = blockIdx.y;
    if (j >= N) return;
    out[l * N + j] = in[l * N + automorph_src(j, log_n, galois)];
}

hks_status launch_automorph(const u64 *in, u64 *out, u32 nlimbs, u32 log_n, u64 galois, cudaStream_t s) {
    const u32 threads = 256;
    const size_t N = (size_t)1 << log_n;
    dim3 grid((u32)((N + threads - 1) / threads), nlimbs);
    ProfScope ps(K_AUTOMORPH, s);
    (void)hks_launch(k_automorph, grid, dim3(threads), 0, s, in, out, log_n, galois);
    HKS_CHECK_LAUNCH();
    ps.done(2.0 * nlimbs * (double)N * 8.0);
    return HKS_OK;
}

// ------------------------------------------------------------------------------------------------
// Fused plaintext-weighted sum (BSGS inner products): each thread owns two
// coefficients of one limb for both ciphertext halves; every weight word is loaded once and used
// for both halves.
__global__ void __launch_bounds__(256) k_pt_wsum(const __grid_constant__ WsumArgs A) {
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << A.log_n;
    const u32 t = blockIdx.y;
    const size_t x = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (x >= N) return;
    const size_t o = (size_t)t * N + x;
    const PrimeConst pc = A.pc[t];
    Acc30 a0[2], a1[2];
    acc_zero(a0[0]); acc_zero(a0[1]);
    acc_zero(a1[0]); acc_zero(a1[1]);
    if (A.accumulate) {   // the running value enters as one more term of weight 1
        const ulonglong2 v0 = *reinterpret_cast<const ulonglong2 *>(A.out0 + o);
        const ulonglong2 v1 = *reinterpret_cast<const ulonglong2 *>(A.out1 + o);
        u32 l, h;
        split30(v0.x, l, h); a0[0].s0 = l; a0[0].s1a = h;
        split30(v0.y, l, h); a0[1].s0 = l; a0[1].s1a = h;
        split30(v1.x, l, h); a1[0].s0 = l; a1[0].s1a = h;
        split30(v1.y, l, h); a1[1].s0 = l; a1[1].s1a = h;
    }
    for (u32 j = 0; j < A.nterm; j++) {
        const ulonglong2 w = *reinterpret_cast<const ulonglong2 *>(A.w[j] + o);
        const ulonglong2 p = *reinterpret_cast<const ulonglong2 *>(A.x0[j] + o);
        const ulonglong2 q = *reinterpret_cast<const ulonglong2 *>(A.x1[j] + o);
        u32 wl, wh, yl, yh;
        split30(w.x, wl, wh);
        split30(p.x, yl, yh); acc_mac(a0[0], yl, yh, wl, wh);
        split30(q.x, yl, yh); acc_mac(a1[0], yl, yh, wl, wh);
        split30(w.y, wl, wh);
        split30(p.y, yl, yh); acc_mac(a0[1], yl, yh, wl, wh);
        split30(q.y, yl, yh); acc_mac(a1[1], yl, yh, wl, wh);
    }
    *reinterpret_cast<ulonglong2 *>(A.out0 + o) = make_ulonglong2(acc_reduce(a0[0], pc), acc_reduce(a0[1], pc));
    *reinterpret_cast<ulonglong2 *>(A.out1 + o) = make_ulonglong2(acc_reduce(a1[0], pc), acc_reduce(a1[1], pc));
}

hks_status launch_pt_wsum(const WsumArgs &a, cudaStream_t s) {
    const u32 threads = 256;
    const size_t N = (size_t)1 << a.log_n;
    dim3 grid((u32)((N / 2 + threads - 1) / threads), a.nlimbs);
    ProfScope ps(K_WSUM, s);
    (void)hks_launch(k_pt_wsum, grid, dim3(threads), 0, s, a);
    HKS_CHECK_LAUNCH();
    ps.done((3.0 * a.nterm + 2.0 + (a.accumulate ? 2.0 : 0.0)) * a.nlimbs * (double)N * 8.0,
            (double)a.nterm * 2.0 * a.nlimbs * (double)N * 4.0);
    return HKS_OK;
}

__global__ void __launch_bounds__(256) k_add_ct(const u64 *__restrict__ r0, const u64 *__restrict__ r1,
                                                u64 *__restrict__ out0, u64 *__restrict__ out1, u32 log_n,
                                                const PrimeConst *__restrict__ pcs) {
    pdl_trigger();
    pdl_wait();
    const size_t N = (size_t)1 << log_n;
    const u32 t = blockIdx.y;
    const size_t x = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (x >= N) return;
    const size_t o = (size_t)t * N + x;
    const u64 p = pcs[t].p;
    const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(r0 + o), b = *reinterpret_cast<const ulonglong2 *>(r1 + o);
    ulonglong2 u = *reinterpret_cast<const ulonglong2 *>(out0 + o), v = *reinterpret_cast<const ulonglong2 *>(out1 + o);
    u.x = csub(u.x + a.x, p); u.y = csub(u.y + a.y, p);
    v.x = csub(v.x + b.x, p); v.y = csub(v.y + b.y, p);
    *reinterpret_cast<ulonglong2 *>(out0 + o) = u;
    *reinterpret_cast<ulonglong2 *>(out1 + o) = v;
}

hks_status launch_add_ct(const u64 *r0, const u64 *r1, u64 *out0, u64 *out1, u32 nlimbs, u32 log_n,
                         const PrimeConst *pc, cudaStream_t s) {
    const u32 threads = 256;
    const size_t N = (size_t)1 << log_n;
    dim3 grid((u32)((N / 2 + threads - 1) / threads), nlimbs);
    ProfScope ps(K_ADD, s);
    (void)hks_launch(k_add_ct, grid, dim3(threads), 0, s, r0, r1, out0, out1, log_n, pc);
    HKS_CHECK_LAUNCH();
    ps.done(6.0 * nlimbs * (double)N * 8.0, 0.0);
    return HKS_OK;
}
