// ntt.cu -- batched negacyclic NTT / INTT for sm_100a (§3.6.4).
//
// Design (B200-first):
//   * A limb of N = R x C words is viewed as R rows of C contiguous words.  The radix-2 transform
//     factors into column stages (strides >= C) and row stages (strides < C), so a limb needs two
//     passes over HBM/L2 ("hierarchical / 2D NTT", four memory accesses per element),
//     each a batched kernel over a limb batch (limb batching).
//   * Forward = Cooley-Tukey with merged psi twiddles, natural COEFF in, bit-reversed EVAL out;
//     inverse = Gentleman-Sande, bit-reversed in, natural out, no bit-reversal pass.
//     Pass order: forward COLS -> ROWS, inverse ROWS -> COLS.
//   * Within a pass a CTA owns a tile of NB sub-transforms (NB columns, or NB rows) of length n.
//     Each thread holds E = 2^LOGE elements in registers and runs LOGE butterfly stages per round
//     (radix-2^LOGE rounds); rounds exchange through padded shared memory.  Global loads/stores are
//     coalesced along the contiguous dimension.
//   * Twiddles (w, w' Shoup companion) are precomputed per prime; rows use a per-row rearranged
//     table so that row r's twiddles psi_brv[(R + r) 2^s + i] are contiguous.  They are read
//     through the read-only path (L1/L2) -- not recomputed on the fly (the opposite of the paper's
//     RTX 4090 trade-off), because on B200 the integer pipe, not L2, is scarce.
//   * Butterflies are Harvey-lazy: forward values live in [0, 4p), inverse in [0, 2p); the last
//     pass canonicalises and applies the fused epilogue (SCALE, MODDOWN; §3.6.5).
#include <algorithm>

#include <cooperative_groups.h>

#include "internal.h"

// L2 window of the context whose NTT pass is being launched (set by launch_ntt_pass / launch_ntt_kip on the
// calling thread; launches are synchronous host code)
static thread_local const cudaAccessPolicyWindow *t_win = nullptr;

#ifndef HKS_NTT_TC_MINLIMBS
#define HKS_NTT_TC_MINLIMBS 0   // smallest column-pass batch sent to the tensor cores
#endif
#ifndef HKS_NTT_TC_INV
#define HKS_NTT_TC_INV 1        // inverse column passes on the tensor cores too
#endif

#ifndef HKS_NTT_INVCOLS_MINB
#define HKS_NTT_INVCOLS_MINB HKS_NTT_MINB   // resident CTAs requested for the inverse column pass (scale epilogue)
#endif

#ifndef HKS_KIP_TMA
#define HKS_KIP_TMA 0     // 1: key rows prefetched into shared memory with 1D bulk copies (measured slower)
#endif
#ifndef HKS_KIP_TWS
#define HKS_KIP_TWS 1     // 1: the CTA's row twiddles staged in shared memory by cp.async issued before griddepcontrol.wait
#endif
#ifndef HKS_KIP_EXTS
#define HKS_KIP_EXTS 0    // 1: the row pass's input rows staged into its shared buffers by cp.async right after
#endif                    //    griddepcontrol.wait (one memory latency with the twiddles instead of a second one)
#ifndef HKS_KIP_XWARP
#define HKS_KIP_XWARP 0   // 1: four warps per CTA at three digits (the extra one joins the key product)
#endif
#ifndef HKS_KIP_PIPE
#define HKS_KIP_PIPE 0    // 1: key words of the next product step loaded before the current step's products
#endif
#ifndef HKS_KIP_LATEWAIT
#define HKS_KIP_LATEWAIT 1   // the staged twiddles are awaited after the row pass's first loads are issued, so the
#endif                       // two memory latencies overlap instead of following each other
#ifndef HKS_KIP_PF
#define HKS_KIP_PF 0      // 1 / 2: phase 2's key lines prefetched into L1 / L2 at the start of the last row round
#endif
#ifndef HKS_KIP_L2PF
#define HKS_KIP_L2PF 0    // 1: the CTA's key rows prefetched into L2 (bulk prefetch) at the start of the row pass
#endif

// One pass over a limb batch.  LOGN = log2 of the sub-transform length n; LOGE = log2 of the
// elements a thread holds (radix-2^LOGE rounds); LOGNB = log2 of the sub-transforms per CTA;
// LOGC = log2 of the row length C (the column stride).  COLS: sub-transforms are columns (stride C);
// else rows (contiguous).  Values between butterflies live in the lazy ranges of modarith.cuh.
#ifndef HKS_NTT_MINB
#define HKS_NTT_MINB 4
#endif
// One tile (NB sub-transforms of limb b) of a pass.  Round 0 reads global memory (forward and
// inverse-column passes) or the tile the inverse-row prologue staged in shared memory.
// Row passes whose tile (data + its NB twiddle rows) still fits HKS_NTT_MINB CTAs per SM stage the twiddle rows
// in shared memory with cp.async issued before griddepcontrol.wait (the per-row tables are context data, 16 bytes
// per twiddle, mostly HBM-resident behind the key stream: their latency otherwise sits inside the butterfly chains)
#ifndef HKS_ROW_TWS
#define HKS_ROW_TWS 0   // 1: measured slower for the stand-alone row passes (8-row tiles, 32 KB per CTA up front)
#endif
#ifndef HKS_INVROW_OPQ
#define HKS_INVROW_OPQ 1  // inverse row passes: butterfly carry-adds on the ALU pipe (modarith.cuh lazy_add)
#endif
#ifndef HKS_KIP_OPQ
#define HKS_KIP_OPQ 0     // the same for the fused kernel's ModDown inverse row pass
#endif
#ifndef HKS_ROW_L2PF
#define HKS_ROW_L2PF 3    // row passes bulk-prefetch their tile's twiddle rows into L2 before griddepcontrol.wait:
#endif                    // 1 inverse, 2 all, 3 forward (ModDown row pass 37.3 -> 35.5 us; the inverse pass loses)
#ifndef HKS_ROW_L2PF_EPI
#define HKS_ROW_L2PF_EPI 1   // the ModDown row pass also prefetches its epilogue operands (acc, c0) into L2
#endif
#ifndef HKS_ROW_WSYNC
#define HKS_ROW_WSYNC 1   // row passes: a row never straddles a warp, so the exchanges between rounds (and the
#endif                    // staged tile load / copy-out, mapped warp by warp) need __syncwarp, not CTA barriers
template <int LOGN, int LOGE, int LOGNB, bool COLS>
constexpr bool row_tws() {
    return HKS_ROW_TWS && !COLS &&
           ((size_t)((1 << LOGN) + ((1 << LOGN) >> LOGE)) * (1 << LOGNB) * 8 + (size_t)(16 << (LOGN + LOGNB))) * HKS_NTT_MINB <=
               220 * 1024;
}

template <int LOGN, int LOGE, int LOGNB, int LOGC, bool COLS, bool FWD, int EPI>
__device__ __forceinline__ void ntt_tile(const NttArgs &A, const u32 b, const u32 tile, u64 *sm, const ulonglong2 *tws) {
    constexpr int n = 1 << LOGN;
    constexpr int E = 1 << LOGE;
    constexpr int NB = 1 << LOGNB;
    constexpr int C = 1 << LOGC;
    constexpr int TPS = n >> LOGE;                    // threads per sub-transform
    constexpr int NT = NB * TPS;                      // threads per CTA
    constexpr int NR = (LOGN + LOGE - 1) / LOGE;      // rounds
    constexpr int ROWPAD = n + (n >> LOGE);
    constexpr int LOG_NLIMB = COLS ? (LOGN + LOGC) : 0;   // log2 N for the column pass
    constexpr bool MD = EPI == EPI_MODDOWN || EPI == EPI_MDTENSOR;   // ModDown-style epilogue
    constexpr bool CIN = EPI == EPI_LAZY_CIN, COUT = EPI == EPI_SCALE_COUT;   // chunked column-pass I/O

    const u32 prime = A.map.prime[b];
    const u32 log_n = COLS ? (u32)LOG_NLIMB : A.log_n;
    const size_t N = (size_t)1 << log_n;
    const NttMod m = make_nttmod(A.pc[prime].p);
    const int tid = threadIdx.x;
    const int bsub = COLS ? (tid & (NB - 1)) : (tid >> (LOGN - LOGE));
    const int tu = COLS ? (tid >> LOGNB) : (tid & (TPS - 1));
    // element j of this thread's sub-transform lives at src_sub[j * JS]
    constexpr int JS = COLS ? C : 1;
    const size_t sub_off = COLS ? (size_t)(tile * NB + bsub) : (size_t)(tile * NB + bsub) * n;
    const u32 ob = MD ? A.map.ob[b] : 0;   // ModDown output-table entry
    u64 *const out_base = MD ? A.outs[ob] : A.out;
    const u64 *__restrict__ src = A.in + (size_t)A.map.sin[b] * N + sub_off;
    u64 *__restrict__ dst = out_base + (size_t)A.map.sout[b] * N + sub_off;
    // chunked layout (COLS only: element j = row j of column sub_off): chunk base + row-in-chunk offset
    const u32 cmask = (1u << A.clog) - 1;
    const u64 *__restrict__ csrc = A.in + ((size_t)A.map.sin[b] << (A.clog + LOGC)) + sub_off;
    u64 *__restrict__ cdst = out_base + ((size_t)A.map.sout[b] << (A.clog + LOGC)) + sub_off;
    auto cidx = [&](int j) -> size_t { return (size_t)((u32)j >> A.clog) * A.cstride + ((size_t)((u32)j & cmask) << LOGC); };
    const ulonglong2 *tw =
        COLS ? A.tw + (size_t)prime * n : (tws ? tws + bsub * n : A.tw + (((size_t)prime << A.log_r) + tile * NB + bsub) * n);

    auto saddr = [&](int k) -> int {
        return COLS ? (k + (k >> LOGE)) * NB + bsub : bsub * ROWPAD + k + (k >> LOGE);
    };
    // warp-private rows: thread tid's sub-transform bsub = tid / TPS lies inside tid's warp, so the warp's
    // rows are the 32 E contiguous tile words [warp * 32 E, (warp + 1) * 32 E)
    constexpr bool WS = HKS_ROW_WSYNC && !COLS && TPS <= 32 && (NT % 32) == 0 && !row_tws<LOGN, LOGE, LOGNB, COLS>();
    auto rsync = [&]() {
        if (WS) __syncwarp(); else __syncthreads();
    };
    // tile word handled by this thread in the q-th coalesced sweep of a staged load / copy-out
    auto tix = [&](int q) -> int { return WS ? ((tid & ~31) * E + (tid & 31) + 32 * q) : (tid + q * NT); };

    // epilogue constants
    ulonglong2 sc = make_ulonglong2(0, 0);
    if (EPI == EPI_SCALE || EPI == EPI_SCALE_COUT) sc = A.scale ? A.scale[b % A.scale_mod] : A.ninv[prime];
    ulonglong2 pinv = make_ulonglong2(0, 0);
    const u64 *ea = nullptr, *eb = nullptr;
    if (MD) {
        if (A.pinv) pinv = A.pinv[prime];
        ea = A.ea + (size_t)A.map.sa[b] * N + sub_off;
        const u64 *ebase = A.adds[ob];
        eb = (EPI == EPI_MODDOWN && ebase && A.map.sb[b] != 0xffff) ? ebase + (size_t)A.map.sb[b] * N : nullptr;
    }
    const u64 galois = MD ? A.ogal[ob] : 1;
    // ModDown core (a - x) P^-1, a canonical, x < 8p + 2^32; A.pinv == NULL: the key was prepared with P^-1 on
    // its Q limbs and P^-1 folded into the conversion matrix (hks_evk_prepare), so (a - x) is already the value
    auto md_sub = [&](u64 a, u64 x) -> u64 {
        const u64 d = a + m.eight_p + m.p - x;   // < 10p
        if (A.pinv) return csub(csub(shoup_approx(d, pinv.x, pinv.y, m.np), m.two_p), m.p);
        return csub(csub(csub(csub(d, m.eight_p), m.four_p), m.two_p), m.p);
    };
    // EPI_SWITCH: the column pass loads the source-modulus COEFF limb and switches it into this prime
    const u64 sw_m = EPI == EPI_SWITCH ? A.sw_qmod[prime] : 0;
    auto epi = [&](u64 x, int j) -> u64 {
        if (EPI == EPI_LAZY || EPI == EPI_TENSOR || EPI == EPI_SWITCH || EPI == EPI_LAZY_CIN) return x;
        if (EPI == EPI_SCALE || EPI == EPI_SCALE_COUT) return csub(csub(shoup_approx(x, sc.x, sc.y, m.np), m.two_p), m.p);
        if (EPI == EPI_CANON) return canon8(x, m);
        // EPI_MODDOWN: (a - x) * P^-1 [+ b], a canonical, x < 8p + 2^32
        u64 r = md_sub(ea[(size_t)j * JS], x);
        if (eb) {
            const u32 xg = (u32)(sub_off + (size_t)j * JS);
            r = csub(r + eb[galois == 1 ? xg : automorph_src(xg, log_n, galois)], m.p);
        }
        return r;
    };

    // inverse ROWS (first inverse pass) reads the tile through shared memory (per-thread elements
    // of its first round are contiguous, so a direct load would not coalesce); loads are batched.
    if (!FWD && !COLS) {
        const u64 *__restrict__ tsrc = A.in + (size_t)A.map.sin[b] * N + (size_t)tile * NB * n;
        if (EPI == EPI_TENSOR) {
            // HMult fusion: the INTT input is the tensor term d2 = in * in2, which the
            // key product also needs in EVAL form, so it is stored once to side (4 pairs at a time)
            const u64 *__restrict__ tsrc2 = A.in2 + (size_t)A.map.sin[b] * N + (size_t)tile * NB * n;
            u64 *__restrict__ tside = A.side + (size_t)A.map.sin[b] * N + (size_t)tile * NB * n;
            const PrimeConst pcb = A.pc[prime];
            constexpr int TC = E < 4 ? E : 4;
#pragma unroll
            for (int q0 = 0; q0 < E; q0 += TC) {
                u64 x1[TC], x2[TC];
#pragma unroll
                for (int q = 0; q < TC; q++) {
                    x1[q] = tsrc[tix(q0 + q)];
                    x2[q] = tsrc2[tix(q0 + q)];
                }
#pragma unroll
                for (int q = 0; q < TC; q++) {
                    const int idx = tix(q0 + q), r = idx >> LOGN, k = idx & (n - 1);
                    const u64 d = mulmod_full(x1[q], x2[q], pcb);
                    tside[idx] = d;
                    sm[r * ROWPAD + k + (k >> LOGE)] = d;
                }
            }
        } else {
            u64 tmp[E];
#pragma unroll
            for (int q = 0; q < E; q++) tmp[q] = tsrc[tix(q)];
#pragma unroll
            for (int q = 0; q < E; q++) {
                const int idx = tix(q), r = idx >> LOGN, k = idx & (n - 1);
                sm[r * ROWPAD + k + (k >> LOGE)] = tmp[q];
            }
        }
        rsync();
    }

    u64 v[E];
#pragma unroll
    for (int rr = 0; rr < NR; rr++) {
        const int s0 = rr * LOGE;
        const int e = (LOGN - s0) < LOGE ? (LOGN - s0) : LOGE;
        const int Ee = 1 << e;
        const int UPT = E >> e;
        const int lstride = FWD ? (LOGN - s0 - e) : s0;   // log2 element spacing inside a unit
        const int lBsz = lstride + e;                       // log2 block size
        const bool from_global = (rr == 0) && (FWD || COLS);
        const bool last = (rr == NR - 1);
        if (rr > 0) rsync();

        // gather
#pragma unroll
        for (int q = 0; q < UPT; q++) {
            const int uid = tu * UPT + q;
            const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
            for (int k = 0; k < Ee; k++) {
                const int j = base + (k << lstride);
                if (EPI == EPI_SWITCH && from_global)
                    v[q * Ee + k] = switch_centered(src[(size_t)j * JS], A.sw_q, sw_m, A.pc[prime]);
                else if (CIN && from_global)
                    v[q * Ee + k] = csrc[cidx(j)];
                else
                    v[q * Ee + k] = from_global ? src[(size_t)j * JS] : sm[saddr(j)];
            }
        }
        // butterflies: twiddle of (stage half-size 2^ltg, element j) is tw[(n + j) >> (ltg + 1)],
        // = tw[(n >> s) + (blk << (lBsz - s)) + ((k << lstride) >> s)] with s = ltg + 1.
#pragma unroll
        for (int q = 0; q < UPT; q++) {
            const int uid = tu * UPT + q;
            const int blk = uid >> lstride;
            const int base = (blk << lBsz) + (uid & ((1 << lstride) - 1));
            (void)base;
#pragma unroll
            for (int l = 0; l < e; l++) {
                const int lt = FWD ? (e - 1 - l) : l;
                const int t = 1 << lt;
                const int sh = lt + lstride + 1;
                const ulonglong2 *twb = tw + (n >> sh) + (blk << (lBsz - sh));
#pragma unroll
                for (int k = 0; k < Ee; k++) {
                    if (k & t) continue;
#ifdef HKS_EXPERIMENT_CONST_TW
                    const ulonglong2 w = make_ulonglong2(m.p - 3 - k, 0x123456789abcull + l);   // timing-only experiment
                    (void)twb;
#else
                    const ulonglong2 w = row_tws<LOGN, LOGE, LOGNB, COLS>() ? twb[(k << lstride) >> sh]   // shared
                                                                           : __ldg(twb + ((k << lstride) >> sh));
#endif
                    if (FWD)
                        ct_lazy(v[q * Ee + k], v[q * Ee + k + t], w.x, w.y, m);
                    else
                        gs_lazy<!COLS && HKS_INVROW_OPQ>(v[q * Ee + k], v[q * Ee + k + t], w.x, w.y, m);
                }
            }
        }
        // scatter
        const bool via_smem_out = last && FWD && !COLS;
        if (!last || via_smem_out) {
            if (rr > 0 || !from_global) rsync();
#pragma unroll
            for (int q = 0; q < UPT; q++) {
                const int uid = tu * UPT + q;
                const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                for (int k = 0; k < Ee; k++) {
                    const int j = base + (k << lstride);
                    sm[saddr(j)] = v[q * Ee + k];
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < UPT; q++) {
                const int uid = tu * UPT + q;
                const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                for (int k = 0; k < Ee; k++) {
                    const int j = base + (k << lstride);
                    if (COUT)
                        cdst[cidx(j)] = epi(v[q * Ee + k], j);
                    else
                        dst[(size_t)j * JS] = epi(v[q * Ee + k], j);
                }
            }
        }
    }
    if (FWD && !COLS) {
        // forward ROWS (last forward pass): coalesced copy-out through shared memory, epilogue here.
        // All global operands of the epilogue are loaded first so their latencies overlap.
        rsync();
        const size_t tbase = (size_t)tile * NB * n;
        u64 *__restrict__ tdst = out_base + (size_t)A.map.sout[b] * N + tbase;
        constexpr int CHM = EPI == EPI_MDTENSOR ? 2 : 8;
        constexpr int CH = E < CHM ? E : CHM;   // epilogue chunk: loads of a chunk are issued together
        const bool role1 = EPI == EPI_MDTENSOR && A.trole[ob] != 0;
        const size_t tso = (size_t)A.map.sout[b] * N + tbase;   // tensor operand slot = output limb
#pragma unroll
        for (int q0 = 0; q0 < E; q0 += CH) {
            u64 av[CH], bv[CH], ta[CH], tb[CH], tc[CH], td[CH];
            if (MD) {
                const u64 *__restrict__ tea = A.ea + (size_t)A.map.sa[b] * N + tbase;
#pragma unroll
                for (int q = 0; q < CH; q++) av[q] = tea[tix(q0 + q)];
                if (EPI == EPI_MDTENSOR) {
#pragma unroll
                    for (int q = 0; q < CH; q++) {
                        const size_t o = tso + tix(q0 + q);
                        ta[q] = A.ta0[o];
                        tb[q] = role1 ? A.tb1[o] : A.tb0[o];
                        if (role1) {
                            tc[q] = A.ta1[o];
                            td[q] = A.tb0[o];
                        }
                    }
                }
                if (eb) {
#pragma unroll
                    for (int q = 0; q < CH; q++) {
                        const u32 xg = (u32)(tbase + tix(q0 + q));
                        bv[q] = eb[galois == 1 ? xg : automorph_src(xg, log_n, galois)];
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < CH; q++) {
                const int idx = tix(q0 + q), r = idx >> LOGN, k = idx & (n - 1);
                u64 x = sm[r * ROWPAD + k + (k >> LOGE)];
                if (EPI == EPI_CANON) {
                    x = canon8(x, m);
                } else if (MD) {
                    u64 rr2 = md_sub(av[q], x);
                    if (eb) rr2 = csub(rr2 + bv[q], m.p);
                    if (EPI == EPI_MDTENSOR) {
                        // HMult: + a0 b0 (role 0) or + a0 b1 + a1 b0 (role 1)
                        const PrimeConst pcb = A.pc[prime];
                        const u64 t = role1 ? mul2mod_full(ta[q], tb[q], tc[q], td[q], pcb) : mulmod_full(ta[q], tb[q], pcb);
                        rr2 = csub(rr2 + t, m.p);
                    }
                    x = rr2;
                }
                tdst[idx] = x;
            }
        }
    }
}

#ifndef HKS_NTT_MINB128
#define HKS_NTT_MINB128 0   // > 0: resident CTAs requested for passes with <= 128 threads per CTA (0: as above)
#endif
template <int LOGN, int LOGE, int LOGNB, int LOGC, bool COLS, bool FWD, int EPI>
__global__ void __launch_bounds__((1 << LOGNB) << (LOGN - LOGE),
                                  (((1 << LOGNB) << (LOGN - LOGE)) >= 512) ? 2
                                  : (HKS_NTT_MINB128 > 0 && ((1 << LOGNB) << (LOGN - LOGE)) <= 128) ? HKS_NTT_MINB128
                                  : (COLS && !FWD) ? HKS_NTT_INVCOLS_MINB : HKS_NTT_MINB)
k_ntt(const __grid_constant__ NttArgs A) {
    extern __shared__ __align__(16) u64 sm[];
    pdl_trigger();
    const u32 b = blockIdx.x / A.tiles, tile = blockIdx.x - b * A.tiles;
    constexpr bool TWS = row_tws<LOGN, LOGE, LOGNB, COLS>();
#if HKS_ROW_L2PF
    if (!COLS && !TWS && (HKS_ROW_L2PF == 2 || (HKS_ROW_L2PF == 1 && !FWD) || (HKS_ROW_L2PF == 3 && FWD)) &&
        threadIdx.x == 0) {
        // this tile's per-row twiddle tables (context data, contiguous) requested into L2 before griddepcontrol.wait
        const ulonglong2 *t = A.tw + (((size_t)A.map.prime[b] << A.log_r) + ((size_t)tile << LOGNB)) * (1 << LOGN);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(t), "r"((u32)(16u << (LOGN + LOGNB))) : "memory");
        if (HKS_ROW_L2PF_EPI && (EPI == EPI_MODDOWN || EPI == EPI_MDTENSOR)) {
            // the ModDown epilogue's accumulator and c0 rows of this tile: L2 is the coherence point, so a prefetch
            // is safe even before griddepcontrol.wait (it moves no data into the SM)
            const size_t N = (size_t)1 << A.log_n, off = ((size_t)tile << LOGNB) << LOGN;
            const u32 bytes = 8u << (LOGN + LOGNB);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.ea + (size_t)A.map.sa[b] * N + off), "r"(bytes)
                         : "memory");
            const u32 ob = A.map.ob[b];
            if (EPI == EPI_MODDOWN && A.adds[ob] && A.map.sb[b] != 0xffff && A.ogal[ob] == 1)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.adds[ob] + (size_t)A.map.sb[b] * N + off),
                             "r"(bytes)
                             : "memory");
        }
    }
#endif
    ulonglong2 *tws = nullptr;
    if (TWS) {
        constexpr int NT = (1 << LOGNB) << (LOGN - LOGE), NE = 1 << (LOGN + LOGNB);
        tws = reinterpret_cast<ulonglong2 *>(sm + (size_t)((1 << LOGN) + ((1 << LOGN) >> LOGE)) * (1 << LOGNB));
        const ulonglong2 *src = A.tw + (((size_t)A.map.prime[b] << A.log_r) + ((size_t)tile << LOGNB)) * (1 << LOGN);
        for (int e = threadIdx.x; e < NE; e += NT)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((u32)__cvta_generic_to_shared(tws + e)), "l"(src + e)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    pdl_wait();
    if (TWS) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    ntt_tile<LOGN, LOGE, LOGNB, LOGC, COLS, FWD, EPI>(A, b, tile, sm, tws);
}

template <int LOGN, int LOGE, int LOGNB, int LOGC, bool COLS, bool FWD, int EPI>
static hks_status go(NttArgs &a, cudaStream_t s) {
    constexpr int threads = (1 << LOGNB) << (LOGN - LOGE);
    constexpr size_t smem = (size_t)((1 << LOGN) + ((1 << LOGN) >> LOGE)) * (1 << LOGNB) * sizeof(u64) +
                            (row_tws<LOGN, LOGE, LOGNB, COLS>() ? (size_t)(16 << (LOGN + LOGNB)) : 0);
    auto kern = k_ntt<LOGN, LOGE, LOGNB, LOGC, COLS, FWD, EPI>;
    if (smem > 48 * 1024) {
        hks_func_smem((const void *)kern, smem);
    }
    a.tiles = COLS ? ((1u << a.log_c) >> LOGNB) : ((1u << a.log_r) >> LOGNB);
    const int cls = FWD ? (COLS ? K_NTT_FWD_COLS : ((EPI == EPI_MODDOWN || EPI == EPI_MDTENSOR) ? K_NTT_FWD_ROWS_MODDOWN : K_NTT_FWD_ROWS))
                        : (COLS ? K_NTT_INV_COLS : K_NTT_INV_ROWS);
    ProfScope ps(cls, s);
    (void)hks_launch_ex(pdl_enabled(), t_win, kern, dim3(a.nlimbs * a.tiles), dim3(threads), smem, s, a);
    HKS_CHECK_LAUNCH();
    // algorithmic bytes: each limb read once and written once (+ ModDown operands acc, c0)
    double words = 2.0 * a.nlimbs;
    if (EPI == EPI_MODDOWN)
        for (u32 i = 0; i < a.nlimbs; i++) words += (a.adds[a.map.ob[i]] && a.map.sb[i] != 0xffff) ? 2.0 : 1.0;
    double tmuls = 0;   // tensor products: 4 partial products each
    if (EPI == EPI_MDTENSOR)
        for (u32 i = 0; i < a.nlimbs; i++) {
            const bool r1 = a.trole[a.map.ob[i]] != 0;
            words += r1 ? 5.0 : 3.0;
            tmuls += r1 ? 8.0 : 4.0;
        }
    if (EPI == EPI_TENSOR) {
        words += 2.0 * a.nlimbs;   // second factor in, product out
        tmuls += 4.0 * a.nlimbs;
    }
    // butterflies of this pass: N/2 per stage, LOGN stages; +1 Shoup per element for SCALE/MODDOWN
    const double nn = (double)(1ull << a.log_n);
    double muls = a.nlimbs * (nn / 2.0) * LOGN * 7.0;
    if (EPI == EPI_SCALE || EPI == EPI_SCALE_COUT || EPI == EPI_MODDOWN || EPI == EPI_MDTENSOR) muls += a.nlimbs * nn * 7.0;
    muls += tmuls * nn;
    ps.done(words * nn * 8.0, muls);
    return HKS_OK;
}

template <int LR, int ER, int BR, int LC, int EC, int BC>
static hks_status dispatch(NttDir dir, bool cols, int epi, NttArgs &a, cudaStream_t s) {
    if (dir == NTT_FWD && cols && epi == EPI_SWITCH) return go<LR, ER, BR, LC, true, true, EPI_SWITCH>(a, s);
    if (dir == NTT_FWD && cols && epi == EPI_LAZY_CIN) return go<LR, ER, BR, LC, true, true, EPI_LAZY_CIN>(a, s);
    if (dir == NTT_FWD && cols) return go<LR, ER, BR, LC, true, true, EPI_LAZY>(a, s);
    if (dir == NTT_FWD && epi == EPI_CANON) return go<LC, EC, BC, LC, false, true, EPI_CANON>(a, s);
    if (dir == NTT_FWD && epi == EPI_MODDOWN) return go<LC, EC, BC, LC, false, true, EPI_MODDOWN>(a, s);
    if (dir == NTT_FWD && epi == EPI_MDTENSOR) return go<LC, EC, BC, LC, false, true, EPI_MDTENSOR>(a, s);
    if (dir == NTT_INV && !cols && epi == EPI_TENSOR) return go<LC, EC, BC, LC, false, false, EPI_TENSOR>(a, s);
    if (dir == NTT_INV && !cols) return go<LC, EC, BC, LC, false, false, EPI_LAZY>(a, s);
    if (dir == NTT_INV && cols && epi == EPI_SCALE_COUT) return go<LR, ER, BR, LC, true, false, EPI_SCALE_COUT>(a, s);
    if (dir == NTT_INV && cols) return go<LR, ER, BR, LC, true, false, EPI_SCALE>(a, s);
    HKS_FAIL(HKS_EINVAL, "ntt: unsupported epilogue %d", epi);
}

// Per ring size: sub-transform shapes (log length, log elements per thread, log sub-transforms per
// CTA) of the column pass (length R) and the row pass (length C).  Batches too small to fill two
// waves of 256-thread CTAs use radix-8 rounds (E = 8, twice the warps per tile) at N = 2^16 / 2^17.
// N = 2^16 pass shapes (log length, log elements per thread, log sub-transforms per CTA) x (cols, rows);
// experiment presets selected with -DHKS_D16_BIG_SEL / -DHKS_D16_SMALL_SEL (nvcc splits -D values at commas)
#if defined(HKS_D16_BIG_SEL) && HKS_D16_BIG_SEL == 1
#define HKS_D16_BIG 8, 5, 4, 8, 5, 4
#elif defined(HKS_D16_BIG_SEL) && HKS_D16_BIG_SEL == 2
#define HKS_D16_BIG 8, 4, 3, 8, 4, 3
#else
#define HKS_D16_BIG 8, 4, 4, 8, 4, 4     // large batches: radix-16 rounds, 16 sub-transforms per CTA
#endif
#if defined(HKS_D16_SMALL_SEL) && HKS_D16_SMALL_SEL == 1
#define HKS_D16_SMALL 8, 4, 3, 8, 4, 3
#elif defined(HKS_D16_SMALL_SEL) && HKS_D16_SMALL_SEL == 2
#define HKS_D16_SMALL 8, 3, 3, 8, 3, 3
#elif defined(HKS_D16_SMALL_SEL) && HKS_D16_SMALL_SEL == 3
#define HKS_D16_SMALL 8, 4, 3, 8, 3, 3
#elif defined(HKS_D16_SMALL_SEL) && HKS_D16_SMALL_SEL == 4
#define HKS_D16_SMALL 8, 4, 3, 8, 3, 2
#elif defined(HKS_D16_SMALL_SEL) && HKS_D16_SMALL_SEL == 5
#define HKS_D16_SMALL 8, 4, 3, 8, 4, 2
#elif defined(HKS_D16_SMALL_SEL) && HKS_D16_SMALL_SEL == 6
#define HKS_D16_SMALL 8, 3, 4, 8, 3, 4   // previous default (radix-8, 16 sub-transforms per CTA both passes)
#else
// small batches (< 74 limbs: the 30-limb INTT, ModDown's 20- and 60-limb passes): columns radix-16 with
// 8 columns per CTA (128 threads, 64-byte row segments), rows radix-8 with 8 rows per CTA (256
// threads) -- measured per pass: C2 3 162 -> 3 298 KS/s over the previous 8,3,4,8,3,4
#define HKS_D16_SMALL 8, 4, 3, 8, 3, 3
#endif
#ifndef HKS_SMALL_LIMIT
#define HKS_SMALL_LIMIT (2u * 148u * 4u)
#endif
hks_status launch_ntt_pass(const hks_ctx *ctx, NttDir dir, int pass, int epi, NttArgs &a, cudaStream_t s) {
    t_win = &ctx->tw_win;
    a.log_n = ctx->log_n;
    a.log_r = ctx->log_r;
    a.log_c = ctx->log_c;
    const bool cols = (dir == NTT_FWD) ? (pass == 0) : (pass == 1);
    if (cols && ctx->log_n == 16 && ctx->all_big && ctx->d_ntt_img_fwd && ntt_tc_enabled() &&
        a.nlimbs >= HKS_NTT_TC_MINLIMBS &&
        ((dir == NTT_FWD && epi == EPI_LAZY) || (HKS_NTT_TC_INV && dir == NTT_INV && epi == EPI_SCALE)))
        return launch_ntt_cols_tc(ctx, dir, epi, a, s);
    const bool small = a.nlimbs * 16u < HKS_SMALL_LIMIT;
    switch (ctx->log_n) {
        case 17: return small ? dispatch<9, 3, 3, 8, 3, 4>(dir, cols, epi, a, s) : dispatch<9, 4, 3, 8, 4, 4>(dir, cols, epi, a, s);
        case 16: return small ? dispatch<HKS_D16_SMALL>(dir, cols, epi, a, s) : dispatch<HKS_D16_BIG>(dir, cols, epi, a, s);
        case 15: return dispatch<8, 4, 4, 7, 4, 4>(dir, cols, epi, a, s);
        case 14: return dispatch<7, 4, 4, 7, 4, 4>(dir, cols, epi, a, s);
        case 13: return dispatch<7, 4, 4, 6, 3, 4>(dir, cols, epi, a, s);
        case 12: return dispatch<6, 3, 4, 6, 3, 4>(dir, cols, epi, a, s);
        case 11: return dispatch<6, 3, 4, 5, 3, 4>(dir, cols, epi, a, s);
        case 10: return dispatch<5, 3, 4, 5, 3, 4>(dir, cols, epi, a, s);
        default: break;
    }
    HKS_FAIL(HKS_EINVAL, "ntt: unsupported log_n %u", ctx->log_n);
}

// ------------------------------------------------------------------------------------------------
// Single-pass inverse NTT at N = 2^16 on a thread-block cluster (§3.6.4: the hierarchical
// NTT reads and writes every element twice; here once).  One cluster of ICL_CS = 4 CTAs per limb; CTA k
// holds rows [64k, 64k + 64) of the 256 x 256 limb in shared memory (139 KB).
//   phase 1: the 8 row stages of its rows (Gentleman-Sande, per-row twiddle table, as the row pass);
//   phase 2: the 6 column stages whose butterflies stay inside its 64 rows (distances 1..32 rows);
//   cluster barrier, then the last two column stages (distances 64 and 128 rows) as one radix-4 step over
//   the four CTAs: CTA k takes columns [64k, 64k + 64) of every row, reads the other CTAs' rows through
//   distributed shared memory, applies the scale epilogue (EPI_SCALE) and writes the natural-order limb.
// The butterflies, their stage order and the lazy arithmetic are those of the two-pass INTT (run_ntt), so
// the output is bit-identical to it.
// Measured: 49.5 us per 30-limb INTT against 21.6 + 19 us for the two passes -- one 1024-thread
// CTA per SM leaves no co-resident CTA to overlap its load, twiddle and exchange latencies -- so it is opt-in.
#ifndef HKS_INTT_CLUSTER
#define HKS_INTT_CLUSTER 0   // 1: the plain INTTs at N = 2^16 in one cluster launch instead of two passes
#endif
#if HKS_INTT_CLUSTER
constexpr int ICL_CS = 4, ICL_ROWS = 64, ICL_N = 256, ICL_PAD = ICL_N + ICL_N / 16, ICL_T = 1024;

// GS stages l < log2 E on v[k] = element j0 + (k << ldj) of a length-n sub-transform: the butterfly at
// distance T = 2^(ldj + l) on element j takes twiddle tw[(n + j) >> (ldj + l + 1)] (see ntt_tile)
template <int E, bool OPQ>
__device__ __forceinline__ void gs_stages(u64 (&v)[E], const ulonglong2 *__restrict__ tw, int n, int j0, int ldj,
                                          const NttMod &m) {
#pragma unroll
    for (int l = 0; (1 << l) < E; l++) {
        const int t = 1 << l;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & t) continue;
            const ulonglong2 w = __ldg(tw + ((n + j0 + (k << ldj)) >> (ldj + l + 1)));
            gs_lazy<OPQ>(v[k], v[k + t], w.x, w.y, m);
        }
    }
}

__global__ void __cluster_dims__(ICL_CS, 1, 1) __launch_bounds__(ICL_T, 1) k_intt_cl(const __grid_constant__ NttArgs A) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) u64 sm[];
    pdl_trigger();
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const u32 b = blockIdx.x / ICL_CS;
    const u32 prime = A.map.prime[b];
    const NttMod m = make_nttmod(A.pc[prime].p);
    const int tid = threadIdx.x;
    const int R0 = rank * ICL_ROWS;
    constexpr size_t NW = (size_t)ICL_N * ICL_N;
    auto sidx = [](int r, int c) { return r * ICL_PAD + c + (c >> 4); };
    const ulonglong2 *__restrict__ twr = A.tw + (((size_t)prime << 8) + R0) * ICL_N;   // this CTA's row tables
    const ulonglong2 *__restrict__ twc = A.tw2 + (size_t)prime * ICL_N;
    if (tid == 0) {
        // context tables (no kernel writes them): this CTA's 64 row tables (256 KB, contiguous) and the column
        // table head for L2 before griddepcontrol.wait, so the row stages' twiddle loads are L2 hits
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(twr), "r"((u32)(ICL_ROWS * ICL_N * 16)) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(twc), "r"((u32)(ICL_N * 16)) : "memory");
    }
    pdl_wait();

    // phase 0: the CTA's rows into shared memory, coalesced and warp by warp (warp w: rows 2w, 2w + 1)
    {
        const u64 *__restrict__ src = A.in + (size_t)A.map.sin[b] * NW + (size_t)R0 * ICL_N + (tid & ~31) * 16 + (tid & 31);
        u64 t[16];
#pragma unroll
        for (int q = 0; q < 16; q++) t[q] = src[32 * q];
#pragma unroll
        for (int q = 0; q < 16; q++) {
            const int x = (tid & ~31) * 16 + (tid & 31) + 32 * q;
            sm[sidx(x >> 8, x & 255)] = t[q];
        }
        __syncwarp();
    }
    // phase 1: row stages; thread = (row r, 16-element unit tu), rows warp-private
    {
        const int r = tid >> 4, tu = tid & 15;
        const ulonglong2 *tw = twr + (size_t)r * ICL_N;
        u64 v[16];
#pragma unroll
        for (int k = 0; k < 16; k++) v[k] = sm[sidx(r, 16 * tu + k)];
        gs_stages<16, HKS_INVROW_OPQ>(v, tw, ICL_N, 16 * tu, 0, m);   // distances 1..8
#pragma unroll
        for (int k = 0; k < 16; k++) sm[sidx(r, 16 * tu + k)] = v[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 16; k++) v[k] = sm[sidx(r, tu + 16 * k)];
        gs_stages<16, HKS_INVROW_OPQ>(v, tw, ICL_N, tu, 4, m);        // distances 16..128
#pragma unroll
        for (int k = 0; k < 16; k++) sm[sidx(r, tu + 16 * k)] = v[k];
    }
    __syncthreads();
    // phase 2a: column stages at row distances 1..8 (thread = column c, rows 16 g .. 16 g + 15), then 16, 32
    {
        const int c = tid & 255, g = tid >> 8;
        u64 v[16];
#pragma unroll
        for (int k = 0; k < 16; k++) v[k] = sm[sidx(16 * g + k, c)];
        gs_stages<16, false>(v, twc, ICL_N, R0 + 16 * g, 0, m);
#pragma unroll
        for (int k = 0; k < 16; k++) sm[sidx(16 * g + k, c)] = v[k];
    }
    __syncthreads();
    {
        const int c = tid & 255, q = tid >> 8;   // row units r0 = 4 q + i (i < 4): rows r0 + 16 jj
        u64 v[4][4];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int jj = 0; jj < 4; jj++) v[i][jj] = sm[sidx(4 * q + i + 16 * jj, c)];
#pragma unroll
        for (int i = 0; i < 4; i++) gs_stages<4, false>(v[i], twc, ICL_N, R0 + 4 * q + i, 4, m);
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int jj = 0; jj < 4; jj++) sm[sidx(4 * q + i + 16 * jj, c)] = v[i][jj];
    }
    cl.sync();   // every CTA's rows have their first 14 stages
    // phase 2b: distances 64 and 128 rows across the cluster; thread = (column c of this CTA's 64, row quad)
    {
        const int c = ICL_ROWS * rank + (tid & 63), rq = tid >> 6;
        const ulonglong2 sc = A.scale ? A.scale[b % A.scale_mod] : A.ninv[prime];
        u64 *__restrict__ dst = A.out + (size_t)A.map.sout[b] * NW + c;
        u64 v[4][4];
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
            u32 ra;   // CTA jj's copy of this shared-memory word (distributed shared memory)
            asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((u32)__cvta_generic_to_shared(sm + sidx(4 * rq, c))), "r"(jj));
#pragma unroll
            for (int i = 0; i < 4; i++)
                asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v[i][jj]) : "r"(ra + (u32)(i * ICL_PAD * 8)) : "memory");
        }
#pragma unroll
        for (int i = 0; i < 4; i++) gs_stages<4, false>(v[i], twc, ICL_N, 4 * rq + i, 6, m);
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int jj = 0; jj < 4; jj++)
                dst[(size_t)(4 * rq + i + ICL_ROWS * jj) * ICL_N] =
                    csub(csub(shoup_approx(v[i][jj], sc.x, sc.y, m.np), m.two_p), m.p);
    }
    cl.sync();   // no CTA exits while another still reads its shared memory
}

static bool intt_cluster_ok(const hks_ctx *ctx) { return ctx->log_n == 16 && ctx->log_r == 8; }

static hks_status launch_intt_cluster(const hks_ctx *ctx, NttArgs &a, cudaStream_t s) {
    constexpr size_t smem = (size_t)ICL_ROWS * ICL_PAD * sizeof(u64);
    hks_func_smem((const void *)k_intt_cl, smem);
    a.log_n = ctx->log_n;
    a.log_r = ctx->log_r;
    a.log_c = ctx->log_c;
    a.tiles = ICL_CS;
    ProfScope ps(K_NTT_INV_FUSED, s);
    (void)hks_launch_ex(pdl_enabled(), &ctx->tw_win, k_intt_cl, dim3(a.nlimbs * ICL_CS), dim3(ICL_T), smem, s, a);
    HKS_CHECK_LAUNCH();
    const double nn = 65536.0;
    // one read and one write per element; 16 stages of N/2 butterflies + one scale product per element
    ps.done(2.0 * a.nlimbs * nn * 8.0, a.nlimbs * ((nn / 2.0) * 16.0 + nn) * 7.0);
    return HKS_OK;
}
#else
static bool intt_cluster_ok(const hks_ctx *) { return false; }
static hks_status launch_intt_cluster(const hks_ctx *, NttArgs &, cudaStream_t) { return HKS_EINVAL; }
#endif

static void fill_map(NttArgs &a, const LimbList &L, size_t off, u32 cnt, bool second_pass) {
    for (u32 i = 0; i < cnt; i++) {
        a.map.sin[i] = second_pass ? L.sout[off + i] : L.sin[off + i];
        a.map.sout[i] = L.sout[off + i];
        a.map.prime[i] = L.prime[off + i];
        a.map.sa[i] = L.sa[off + i];
        a.map.sb[i] = L.sb[off + i];
        a.map.ob[i] = 0;
    }
    a.nlimbs = cnt;
}

hks_status run_ntt(const hks_ctx *ctx, NttDir dir, const LimbList &L, const u64 *in, u64 *out,
                   const ulonglong2 *scale, u32 scale_mod, cudaStream_t s, const u64 *in2, u64 *side) {
    if (in2 && dir != NTT_INV) HKS_FAIL(HKS_EINVAL, "ntt: tensor prologue only on the inverse transform");
    for (size_t off = 0; off < L.size(); off += HKS_MAXB) {
        u32 cnt = (u32)((L.size() - off) < HKS_MAXB ? (L.size() - off) : HKS_MAXB);
        NttArgs a{};
        a.pc = ctx->d_pc;
        a.ninv = ctx->d_ninv;
        a.galois = 1;
        // pass 0
        fill_map(a, L, off, cnt, false);
        a.in = in;
        a.out = out;
        if (dir == NTT_INV && !in2 && intt_cluster_ok(ctx)) {   // both passes in one cluster launch
            a.tw = ctx->d_tw_row_inv;
            a.tw2 = ctx->d_tw_col_inv;
            a.scale = scale;
            a.scale_mod = scale_mod ? scale_mod : 1;
            if (scale && off != 0) {
                hks_set_error("ntt: scaled batch larger than one launch");
                return HKS_EINVAL;
            }
            hks_status st = launch_intt_cluster(ctx, a, s);
            if (st != HKS_OK) return st;
            continue;
        }
        a.tw = dir == NTT_FWD ? ctx->d_tw_col_fwd : ctx->d_tw_row_inv;
        a.in2 = in2;
        a.side = side;
        hks_status st = launch_ntt_pass(ctx, dir, 0, in2 ? EPI_TENSOR : EPI_LAZY, a, s);
        if (st != HKS_OK) return st;
        // pass 1 (in place on out)
        fill_map(a, L, off, cnt, true);
        a.in = out;
        a.tw = dir == NTT_FWD ? ctx->d_tw_row_fwd : ctx->d_tw_col_inv;
        a.scale = scale;
        a.scale_mod = scale_mod ? scale_mod : 1;
        if (scale && off != 0) {
            hks_set_error("ntt: scaled batch larger than one launch");
            return HKS_EINVAL;
        }
        st = launch_ntt_pass(ctx, dir, 1, dir == NTT_FWD ? EPI_CANON : EPI_SCALE, a, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}

hks_status run_ntt_fwd_cols(const hks_ctx *ctx, const LimbList &L, const u64 *in, u64 *out, cudaStream_t s) {
    for (size_t off = 0; off < L.size(); off += HKS_MAXB) {
        u32 cnt = (u32)((L.size() - off) < HKS_MAXB ? (L.size() - off) : HKS_MAXB);
        NttArgs a{};
        a.pc = ctx->d_pc;
        a.ninv = ctx->d_ninv;
        a.galois = 1;
        fill_map(a, L, off, cnt, false);
        a.in = in;
        a.out = out;
        a.tw = ctx->d_tw_col_fwd;
        hks_status st = launch_ntt_pass(ctx, NTT_FWD, 0, EPI_LAZY, a, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}

hks_status run_ntt_inv_cols(const hks_ctx *ctx, const LimbList &L, const u64 *in, u64 *out, const ulonglong2 *scale,
                            u32 scale_mod, cudaStream_t s) {
    if (L.size() > HKS_MAXB) HKS_FAIL(HKS_EINVAL, "ntt: scaled batch larger than one launch");
    NttArgs a{};
    a.pc = ctx->d_pc;
    a.ninv = ctx->d_ninv;
    a.galois = 1;
    fill_map(a, L, 0, (u32)L.size(), false);
    a.in = in;
    a.out = out;
    a.tw = ctx->d_tw_col_inv;
    a.scale = scale;
    a.scale_mod = scale_mod ? scale_mod : 1;
    return launch_ntt_pass(ctx, NTT_INV, 1, EPI_SCALE, a, s);
}

hks_status run_ntt_moddown(const hks_ctx *ctx, const LimbList &L, const std::vector<uint8_t> &poly,
                           const std::vector<MdOut> &outs, u64 *buf, const u64 *acc, cudaStream_t s,
                           const u64 *const *tensor, const ChunkIn *cin, bool prepared) {
    size_t off = 0;
    while (off < L.size()) {
        // one launch: at most HKS_MAXB limbs spanning at most NTT_MAXO polynomials
        size_t end = off;
        std::vector<uint8_t> seen;
        while (end < L.size() && end - off < HKS_MAXB) {
            const uint8_t p = poly[end];
            if (std::find(seen.begin(), seen.end(), p) == seen.end()) {
                if (seen.size() == NTT_MAXO) break;
                seen.push_back(p);
            }
            end++;
        }
        const u32 cnt = (u32)(end - off);
        NttArgs a{};
        a.pc = ctx->d_pc;
        a.ninv = ctx->d_ninv;
        a.pinv = prepared ? nullptr : ctx->d_pinv;
        a.galois = 1;
        // pass 0: columns, in place on buf (slots sin) -- or from the chunked input
        for (u32 i = 0; i < cnt; i++) {
            a.map.sin[i] = cin ? cin->slot[off + i] : L.sin[off + i];
            a.map.sout[i] = L.sin[off + i];
            a.map.prime[i] = L.prime[off + i];
        }
        a.nlimbs = cnt;
        a.in = cin ? cin->buf : buf;
        a.out = buf;
        a.tw = ctx->d_tw_col_fwd;
        if (cin) {
            a.clog = cin->clog;
            a.cstride = cin->cstride;
        }
        hks_status st = launch_ntt_pass(ctx, NTT_FWD, 0, cin ? EPI_LAZY_CIN : EPI_LAZY, a, s);
        a.clog = 0;
        a.cstride = 0;
        if (st != HKS_OK) return st;
        // pass 1: rows, buf -> outs[...] with the ModDown epilogue
        fill_map(a, L, off, cnt, false);
        for (u32 k = 0; k < seen.size(); k++) {
            a.outs[k] = outs[seen[k]].out;
            a.adds[k] = outs[seen[k]].add;
            a.ogal[k] = outs[seen[k]].galois;
        }
        for (u32 i = 0; i < cnt; i++)
            a.map.ob[i] = (uint8_t)(std::find(seen.begin(), seen.end(), poly[off + i]) - seen.begin());
        a.in = buf;
        a.ea = acc;
        a.tw = ctx->d_tw_row_fwd;
        if (tensor) {   // HMult: polynomial p of the pair takes tensor role p
            a.ta0 = tensor[0];
            a.ta1 = tensor[1];
            a.tb0 = tensor[2];
            a.tb1 = tensor[3];
            for (u32 k = 0; k < seen.size(); k++) a.trole[k] = seen[k];
        }
        st = launch_ntt_pass(ctx, NTT_FWD, 1, tensor ? EPI_MDTENSOR : EPI_MODDOWN, a, s);
        if (st != HKS_OK) return st;
        off = end;
    }
    return HKS_OK;
}

// Rescale ("Rescale fusion"): for npoly polynomials x_p [l+1][N] EVAL whose top limb
// is already COEFF in coef slot p, out_p[i] = q_l^-1 (x_p[i] - NTT_{q_i}(SwitchModulo(coef_p))) for
// i < l.  Column pass: SwitchModulo fused into the load, into buf slot p*l + i.  Row pass: NTT and
// the epilogue (EPI_MODDOWN with q_l^-1 in place of P^-1).
hks_status run_rescale(const hks_ctx *ctx, u32 npoly, u32 level, const u64 *x, const u64 *coef, u64 *buf,
                       u64 *const *outs, cudaStream_t s) {
    const u32 pl = std::max<u32>(1, std::min<u32>(NTT_MAXO, HKS_MAXB / level));   // polys per launch
    for (u32 p0 = 0; p0 < npoly; p0 += pl) {
        const u32 np_ = std::min(pl, npoly - p0);
        NttArgs a{};
        a.pc = ctx->d_pc;
        a.ninv = ctx->d_ninv;
        a.galois = 1;
        u32 cnt = 0;
        for (u32 p = 0; p < np_; p++)
            for (u32 i = 0; i < level; i++, cnt++) {
                a.map.sin[cnt] = (u16)(p0 + p);
                a.map.sout[cnt] = (u16)((p0 + p) * level + i);
                a.map.prime[cnt] = (u16)i;
            }
        a.nlimbs = cnt;
        a.in = coef;
        a.out = buf;
        a.tw = ctx->d_tw_col_fwd;
        a.sw_q = ctx->primes[level];
        a.sw_qmod = ctx->d_qmod + (size_t)level * ctx->nq;
        hks_status st = launch_ntt_pass(ctx, NTT_FWD, 0, EPI_SWITCH, a, s);
        if (st != HKS_OK) return st;
        cnt = 0;
        for (u32 p = 0; p < np_; p++) {
            a.outs[p] = outs[p0 + p];
            a.adds[p] = nullptr;
            a.ogal[p] = 1;
            for (u32 i = 0; i < level; i++, cnt++) {
                a.map.sin[cnt] = (u16)((p0 + p) * level + i);
                a.map.sout[cnt] = (u16)i;
                a.map.sa[cnt] = (u16)((p0 + p) * (level + 1) + i);
                a.map.sb[cnt] = 0xffff;
                a.map.ob[cnt] = (uint8_t)p;
            }
        }
        a.in = buf;
        a.ea = x;
        a.pinv = ctx->d_qlinv + (size_t)level * ctx->nq;
        a.tw = ctx->d_tw_row_fwd;
        st = launch_ntt_pass(ctx, NTT_FWD, 1, EPI_MODDOWN, a, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}

// ------------------------------------------------------------------------------------------------
// Fused forward row pass + key inner product.  CTA = NB rows of one output limb u.  Phase 1: for
// every digit j whose D_j[u] still needs its row pass, run the row rounds into shared buffer j
// (lazy values).  Phase 2: coalesced sweep over the tile, two coefficients per thread:
// acc_p = sum_j canon(D_j) * evk_j[p] with the 30-bit-split IMAD.WIDE accumulation (one reduction
// per output).  D never returns to HBM.
// resident CTAs per SM requested from ptxas: an 80-register budget per thread (the kernel's natural
// size), 1..16 CTAs
#ifndef HKS_KIP_REGS
#define HKS_KIP_REGS 80   // register budget per thread of the fused row pass + key product
#endif
constexpr int kip_minb(int threads) {
    return (65536 / (HKS_KIP_REGS * threads)) < 1
               ? 1
               : ((65536 / (HKS_KIP_REGS * threads)) > 16 ? 16 : 65536 / (HKS_KIP_REGS * threads));
}
#ifdef KIP_TRACE
__device__ long long g_kip_trace[8192 * 12];
extern "C" void *hks_debug_kip_trace() {
    void *p = nullptr;
    cudaGetSymbolAddress(&p, g_kip_trace);
    return p;
}
#define KIP_T(ev) do { if (threadIdx.x == 0 && blockIdx.x < 8192) g_kip_trace[blockIdx.x * 12 + (ev)] = (ev) == 5 ? (long long)smid() : clock64(); } while (0)
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
#else
#define KIP_T(ev) do { } while (0)
#endif
template <int LOGN, int LOGE, int LOGNB, int NTR, int NDIG>
__global__ void __launch_bounds__(NTR * ((1 << LOGNB) << (LOGN - LOGE)),
                                  kip_minb(NTR * ((1 << LOGNB) << (LOGN - LOGE))))
k_ntt_kip(const __grid_constant__ FusedKipArgs A) {
    pdl_trigger();
    KIP_T(0);
    KIP_T(5);
    constexpr int n = 1 << LOGN;
    constexpr int E = 1 << LOGE;
    constexpr int NB = 1 << LOGNB;
    constexpr int TPS = n >> LOGE;
    constexpr int NTG = NB * TPS;                      // threads per term group
    constexpr int NT = NTR * NTG;                      // threads per CTA
    constexpr int NR = (LOGN + LOGE - 1) / LOGE;
    constexpr int ROWPAD = n + (n >> LOGE);
    constexpr int BUF = NB * ROWPAD;
    // thread groups are whole warps and rows never straddle a warp: the row rounds of phases 1 and 3
    // exchange through warp-private shared rows, so __syncwarp orders them (HKS_ROW_WSYNC)
    constexpr bool KWS = HKS_ROW_WSYNC && (NTG % 32) == 0 && TPS <= 32 && !HKS_KIP_EXTS;
    auto gsync = [&]() {
        if (KWS) __syncwarp(); else __syncthreads();
    };
    extern __shared__ __align__(16) u64 sm[];

    const u32 u = blockIdx.x / A.tiles;
    const u32 tile = blockIdx.x - u * A.tiles;
    const u32 prime = A.map.prime[u];
    const size_t N = (size_t)1 << A.log_n;
    const PrimeConst pc = A.pc[prime];
    const NttMod m = make_nttmod(pc.p);
    const int tid = threadIdx.x;
    const size_t tbase = (size_t)tile * NB * n;
    const size_t kst = (size_t)A.nkey * N;
    const u64 *__restrict__ kbase = A.evk + (size_t)A.map.kslot[u] * N + tbase;
#if HKS_KIP_TWS
    // the NB twiddle rows of this tile (contiguous in the per-row table) -> shared memory, issued before
    // griddepcontrol.wait: context tables, so their HBM latency overlaps the predecessor's tail
    ulonglong2 *stw = reinterpret_cast<ulonglong2 *>(sm + NTR * BUF + (HKS_KIP_TMA ? 2 * NDIG * NB * n : 0));
    auto stage_tw = [&](const ulonglong2 *g) {
        const ulonglong2 *src = g + (((size_t)prime << A.log_r) + tile * NB) * n;
        for (int e = tid; e < NB * n; e += NT)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((u32)__cvta_generic_to_shared(stw + e)),
                         "l"(src + e)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage_tw(A.tw);
#endif
#if HKS_KIP_TMA
    // The key rows of this CTA (2 NDIG contiguous runs of NB n words) stream into shared memory with 1D
    // bulk copies issued before griddepcontrol.wait -- the key is a caller input that no kernel of the
    // chain writes -- so the dominant HBM stream overlaps the predecessor's tail and this CTA's row pass.
    u64 *skey = sm + NTR * BUF;
    __shared__ __align__(8) u64 kbar;
    if (tid == 0) {
        const u32 bar = (u32)__cvta_generic_to_shared(&kbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        constexpr u32 bytes = (u32)(NB * n * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * NDIG * bytes)
                     : "memory");
#pragma unroll
        for (int i = 0; i < NDIG; i++) {
            const u32 j = A.map.dig[u][i];
#pragma unroll
            for (int pp = 0; pp < 2; pp++) {
                const u32 dst = (u32)__cvta_generic_to_shared(skey + (size_t)(2 * i + pp) * NB * n);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                    "l"(kbase + (size_t)(2 * j + pp) * kst), "r"(bytes), "r"(bar)
                    : "memory");
            }
        }
    }
#endif
    pdl_wait();
#if HKS_KIP_EXTS
    {
        const int nw = (int)A.map.ntr[u] * NB * n;
        for (int e = tid; e < nw; e += NT) {
            const int i = e / (NB * n), rem = e - i * (NB * n), bs = rem >> LOGN, jj = rem & (n - 1);
            const u64 *g = A.ext + (size_t)(A.map.dsrc[u][i] & 0x7fff) * N + tbase + rem;
            const u32 d = (u32)__cvta_generic_to_shared(sm + i * BUF + bs * ROWPAD + jj + (jj >> LOGE));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(g) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
#endif
#if HKS_KIP_L2PF
    if (tid == 0)
        for (int i = 0; i < NDIG; i++)
            for (int pp = 0; pp < 2; pp++)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kbase + (size_t)(2 * A.map.dig[u][i] + pp) * kst),
                             "r"((u32)(NB * n * 8))
                             : "memory");
#endif
#if (HKS_KIP_TWS || HKS_KIP_EXTS) && !(HKS_KIP_LATEWAIT && HKS_KIP_TWS && !HKS_KIP_EXTS)
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#endif
    KIP_T(1);

#if HKS_KIP_PIPE
    ulonglong2 kbn[NDIG], kan[NDIG];
#if HKS_KIP_PIPE == 2
    // the first product step's key words are requested before the row pass (the key is a caller input)
    if (2 * tid < NB * n)
#pragma unroll
        for (int i = 0; i < NDIG; i++) {
            const u32 j = A.map.dig[u][i];
            kbn[i] = *reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j) * kst + 2 * tid);
            kan[i] = *reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j + 1) * kst + 2 * tid);
        }
#endif
#endif
    // phase 1: thread group i runs the row pass of term i (< NTR) into shared buffer i, concurrently
    {
        const int i = tid / NTG, gt = tid - i * NTG;
        const int bsub = gt >> (LOGN - LOGE);
        const int tu = gt & (TPS - 1);
#if HKS_KIP_TWS
        const ulonglong2 *tw = stw + bsub * n;
#else
        const ulonglong2 *__restrict__ tw = A.tw + (((size_t)prime << A.log_r) + tile * NB + bsub) * n;
#endif
        u64 *smj = sm + i * BUF + bsub * ROWPAD;
        const bool work = i < (int)A.map.ntr[u];                   // warp-uniform (groups are whole warps)
        const u64 *__restrict__ src = A.ext + (size_t)(A.map.dsrc[u][i] & 0x7fff) * N + tbase + (size_t)bsub * n;
        u64 v[E];
#pragma unroll
        for (int rr = 0; rr < NR; rr++) {
            const int s0 = rr * LOGE;
            const int e = (LOGN - s0) < LOGE ? (LOGN - s0) : LOGE;
            const int Ee = 1 << e;
            const int UPT = E >> e;
            const int lstride = LOGN - s0 - e;
            const int lBsz = lstride + e;
#if HKS_KIP_PF
            if (rr == NR - 1) {
                // phase 2's key rows (2 NDIG runs of NB n words) requested into L1 (1) / L2 (2) one round
                // before the product: one 128-byte line per request, spread over the CTA's threads
                constexpr int LINES = NB * n * 8 / 128;
                for (int e2 = tid; e2 < 2 * NDIG * LINES; e2 += NT) {
                    const int run = e2 / LINES, ln = e2 - run * LINES;
                    const u64 *a = kbase + (size_t)(2 * A.map.dig[u][run >> 1] + (run & 1)) * kst + ln * 16;
                    if (HKS_KIP_PF == 1)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
                    else
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                }
            }
#endif
            if (rr > 0) gsync();
            if (work) {
#pragma unroll
            for (int q = 0; q < UPT; q++) {
                const int uid = tu * UPT + q;
                const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                for (int k = 0; k < Ee; k++) {
                    const int jj = base + (k << lstride);
                    v[q * Ee + k] = (rr == 0 && !HKS_KIP_EXTS) ? src[jj] : smj[jj + (jj >> LOGE)];
                }
            }
#if HKS_KIP_LATEWAIT && HKS_KIP_TWS && !HKS_KIP_EXTS
            }
            if (rr == 0) {   // the staged twiddle rows, awaited after the round-0 loads were issued
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncthreads();
            }
            if (work) {
#endif
#ifdef KIP_TRACE
            if (threadIdx.x == 0 && blockIdx.x < 8192) {   // first use of the gathered values
                u64 acc = 0;
#pragma unroll
                for (int q = 0; q < E; q++) acc ^= v[q];
                g_kip_trace[blockIdx.x * 12 + 6 + 3 * rr] = clock64() + (long long)(acc & 1) * 0;
                asm volatile("" ::"l"(acc));
            }
#endif
#pragma unroll
            for (int q = 0; q < UPT; q++) {
                const int uid = tu * UPT + q;
                const int blk = uid >> lstride;
#pragma unroll
                for (int l = 0; l < e; l++) {
                    const int lt = e - 1 - l;
                    const int t = 1 << lt;
                    const int sh = lt + lstride + 1;
                    const ulonglong2 *twb = tw + (n >> sh) + (blk << (lBsz - sh));
#pragma unroll
                    for (int k = 0; k < Ee; k++) {
                        if (k & t) continue;
#if HKS_KIP_TWS
                        const ulonglong2 w = twb[(k << lstride) >> sh];
#else
                        const ulonglong2 w = __ldg(twb + ((k << lstride) >> sh));
#endif
                        ct_lazy(v[q * Ee + k], v[q * Ee + k + t], w.x, w.y, m);
                    }
                }
            }
#ifdef KIP_TRACE
            if (threadIdx.x == 0 && blockIdx.x < 8192) {
                u64 acc = 0;
#pragma unroll
                for (int q = 0; q < E; q++) acc ^= v[q];
                asm volatile("" ::"l"(acc));
                g_kip_trace[blockIdx.x * 12 + 7 + 3 * rr] = clock64();
            }
#endif
            }
            if (rr > 0 || HKS_KIP_EXTS) gsync();
#ifdef KIP_TRACE
            if (threadIdx.x == 0 && blockIdx.x < 8192) g_kip_trace[blockIdx.x * 12 + 8 + 3 * rr] = clock64();
#endif
            if (work)
#pragma unroll
            for (int q = 0; q < UPT; q++) {
                const int uid = tu * UPT + q;
                const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                for (int k = 0; k < Ee; k++) {
                    const int jj = base + (k << lstride);
                    smj[jj + (jj >> LOGE)] = v[q * Ee + k];
                }
            }
        }
    }
    __syncthreads();
    KIP_T(2);
#if HKS_KIP_TWS
    if (A.map.yslot[u] != 0xffff && NTR >= 2) stage_tw(A.tw_inv);   // phase 3's inverse twiddles, under phase 2
#endif

    // phase 2: acc_p = sum_i canon(D_i) * evk_{dig(i)}[p], two coefficients per thread per step; the
    // loads of all terms are issued before the multiply-accumulates.
#if HKS_KIP_TMA
    {
        const u32 bar = (u32)__cvta_generic_to_shared(&kbar);
        asm volatile("{\n\t.reg .pred p;\n\tKW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra KW%=;\n\t}" ::"r"(bar)
                     : "memory");
    }
#endif
    const u32 as = A.map.aslot[u];
    const u32 ys = A.map.yslot[u];
    const bool ymode = ys != 0xffff && NTR >= 2;      // uniform per CTA
#if HKS_KIP_PIPE
    // key words of step idx (the dominant HBM stream): loaded one step ahead of the products that use them
    auto load_keys = [&](int idx, ulonglong2 (&kb)[NDIG], ulonglong2 (&ka)[NDIG]) {
#pragma unroll
        for (int i = 0; i < NDIG; i++) {
            const u32 j = A.map.dig[u][i];
            kb[i] = *reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j) * kst + idx);
            ka[i] = *reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j + 1) * kst + idx);
        }
    };
#if HKS_KIP_PIPE == 1
    if (2 * tid < NB * n) load_keys(2 * tid, kbn, kan);
#endif
#endif
    for (int idx = 2 * tid; idx < NB * n; idx += 2 * NT) {
        const int r = idx >> LOGN, k = idx & (n - 1);
        ulonglong2 kb[NDIG], ka[NDIG], dv[NDIG];
#if HKS_KIP_PIPE
#pragma unroll
        for (int i = 0; i < NDIG; i++) {
            kb[i] = kbn[i];
            ka[i] = kan[i];
        }
        if (idx + 2 * NT < NB * n) load_keys(idx + 2 * NT, kbn, kan);
#endif
#pragma unroll
        for (int i = 0; i < NDIG; i++) {
            const u32 j = A.map.dig[u][i];
#if HKS_KIP_PIPE
            (void)j;
#elif HKS_KIP_TMA
            (void)j;
            kb[i] = *reinterpret_cast<const ulonglong2 *>(skey + (size_t)(2 * i) * NB * n + idx);
            ka[i] = *reinterpret_cast<const ulonglong2 *>(skey + (size_t)(2 * i + 1) * NB * n + idx);
#else
#if HKS_KEY_STREAM
            // each key word is read once per KeySwitch: streaming hint (evict first) keeps it from evicting
            // the twiddle tables and the ModUp output in L2
            kb[i] = __ldcs(reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j) * kst + idx));
            ka[i] = __ldcs(reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j + 1) * kst + idx));
#else
            kb[i] = *reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j) * kst + idx);
            ka[i] = *reinterpret_cast<const ulonglong2 *>(kbase + (size_t)(2 * j + 1) * kst + idx);
#endif
#endif
            if (i >= (int)A.map.ntr[u]) {
                dv[i] = *reinterpret_cast<const ulonglong2 *>(A.c1 + (size_t)(A.map.dsrc[u][i] & 0x7fff) * N + tbase + idx);
            } else {
                const u64 *smj = sm + i * BUF + r * ROWPAD + k + (k >> LOGE);
                dv[i].x = canon8(smj[0], m);
                dv[i].y = canon8(smj[1], m);
            }
        }
#if HKS_KIP_KARA
        // Karatsuba products (3 IMAD.WIDE each): D split once per term, shared by the two key words
        AccK a0[2], a1[2];
#pragma unroll
        for (int i = 0; i < NDIG; i++) {
            u32 dl, dh, ml, mh;
#define KKP(I)                                                                                    \
            if (i == I) {                                                                         \
                split30(dv[I].x, dl, dh);                                                         \
                u32 ds = dl + dh;                                                                 \
                split30(kb[I].x, ml, mh); acck_mac<I>(a0[0], dl, dh, ds, ml, mh, ml + mh);        \
                split30(ka[I].x, ml, mh); acck_mac<I>(a1[0], dl, dh, ds, ml, mh, ml + mh);        \
                split30(dv[I].y, dl, dh);                                                         \
                ds = dl + dh;                                                                     \
                split30(kb[I].y, ml, mh); acck_mac<I>(a0[1], dl, dh, ds, ml, mh, ml + mh);        \
                split30(ka[I].y, ml, mh); acck_mac<I>(a1[1], dl, dh, ds, ml, mh, ml + mh);        \
            }
            KKP(0) KKP(1) KKP(2) KKP(3)
#undef KKP
        }
        ulonglong2 o0, o1;
        {
            u64 lo, hi;
            acck_to128(a0[0], NDIG, lo, hi); o0.x = reduce128(lo, hi, pc);
            acck_to128(a0[1], NDIG, lo, hi); o0.y = reduce128(lo, hi, pc);
            acck_to128(a1[0], NDIG, lo, hi); o1.x = reduce128(lo, hi, pc);
            acck_to128(a1[1], NDIG, lo, hi); o1.y = reduce128(lo, hi, pc);
        }
#else
        Acc30 a0[2], a1[2];
#pragma unroll
        for (int i = 0; i < NDIG; i++) {
            u32 dl, dh, ml, mh;
            split30(dv[i].x, dl, dh);
            split30(kb[i].x, ml, mh);
            if (i == 0) acc_first(a0[0], dl, dh, ml, mh); else acc_mac(a0[0], dl, dh, ml, mh);
            split30(ka[i].x, ml, mh);
            if (i == 0) acc_first(a1[0], dl, dh, ml, mh); else acc_mac(a1[0], dl, dh, ml, mh);
            split30(dv[i].y, dl, dh);
            split30(kb[i].y, ml, mh);
            if (i == 0) acc_first(a0[1], dl, dh, ml, mh); else acc_mac(a0[1], dl, dh, ml, mh);
            split30(ka[i].y, ml, mh);
            if (i == 0) acc_first(a1[1], dl, dh, ml, mh); else acc_mac(a1[1], dl, dh, ml, mh);
        }
        ulonglong2 o0, o1;
        o0.x = acc_reduce(a0[0], pc);
        o0.y = acc_reduce(a0[1], pc);
        o1.x = acc_reduce(a1[0], pc);
        o1.y = acc_reduce(a1[1], pc);
#endif
        if (ymode) {
            // each thread overwrites only the positions it read its D values from: no race
            u64 *s0 = sm + r * ROWPAD + k + (k >> LOGE);
            s0[0] = o0.x;
            s0[1] = o0.y;
            s0[BUF] = o1.x;
            s0[BUF + 1] = o1.y;
        } else {
            *reinterpret_cast<ulonglong2 *>(A.acc + (size_t)as * N + tbase + idx) = o0;
            *reinterpret_cast<ulonglong2 *>(A.acc + ((size_t)A.acc_stride + as) * N + tbase + idx) = o1;
        }
    }
    KIP_T(3);
    KIP_T(4);
    if (!ymode) return;

    // phase 3 (P limbs): ModDown's first inverse-NTT pass (Gentleman-Sande row stages) on acc_0 / acc_1,
    // thread groups 0 and 1, written to y; the column pass follows in run_ntt_inv_cols.
    __syncthreads();
    {
        const int g = tid / NTG, gt = tid - g * NTG;
        const bool work = g < 2;
        const int bsub = gt >> (LOGN - LOGE);
        const int tu = gt & (TPS - 1);
#if HKS_KIP_TWS
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        const ulonglong2 *tw = stw + bsub * n;
#else
        const ulonglong2 *__restrict__ tw = A.tw_inv + (((size_t)prime << A.log_r) + tile * NB + bsub) * n;
#endif
        u64 *smj = sm + (work ? g : 0) * BUF + bsub * ROWPAD;
        u64 *__restrict__ dst = A.y + ((size_t)(work ? g : 0) * A.ystride + ys) * N + tbase + (size_t)bsub * n;
        u64 v[E];
#pragma unroll
        for (int rr = 0; rr < NR; rr++) {
            const int s0 = rr * LOGE;
            const int e = (LOGN - s0) < LOGE ? (LOGN - s0) : LOGE;
            const int Ee = 1 << e;
            const int UPT = E >> e;
            const int lstride = s0;
            const int lBsz = lstride + e;
            const bool last = rr == NR - 1;
            if (rr > 0) gsync();
            if (work) {
#pragma unroll
                for (int q = 0; q < UPT; q++) {
                    const int uid = tu * UPT + q;
                    const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                    for (int k = 0; k < Ee; k++) {
                        const int jj = base + (k << lstride);
                        v[q * Ee + k] = smj[jj + (jj >> LOGE)];
                    }
                }
#pragma unroll
                for (int q = 0; q < UPT; q++) {
                    const int uid = tu * UPT + q;
                    const int blk = uid >> lstride;
#pragma unroll
                    for (int l = 0; l < e; l++) {
                        const int t = 1 << l;
                        const int sh = l + lstride + 1;
                        const ulonglong2 *twb = tw + (n >> sh) + (blk << (lBsz - sh));
#pragma unroll
                        for (int k = 0; k < Ee; k++) {
                            if (k & t) continue;
#if HKS_KIP_TWS
                            const ulonglong2 w = twb[(k << lstride) >> sh];
#else
                            const ulonglong2 w = __ldg(twb + ((k << lstride) >> sh));
#endif
                            gs_lazy<HKS_KIP_OPQ>(v[q * Ee + k], v[q * Ee + k + t], w.x, w.y, m);
                        }
                    }
                }
            }
            if (!last) {
                gsync();
                if (work) {
#pragma unroll
                    for (int q = 0; q < UPT; q++) {
                        const int uid = tu * UPT + q;
                        const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                        for (int k = 0; k < Ee; k++) {
                            const int jj = base + (k << lstride);
                            smj[jj + (jj >> LOGE)] = v[q * Ee + k];
                        }
                    }
                }
            } else if (work) {
#pragma unroll
                for (int q = 0; q < UPT; q++) {
                    const int uid = tu * UPT + q;
                    const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                    for (int k = 0; k < Ee; k++) dst[base + (k << lstride)] = v[q * Ee + k];
                }
            }
        }
    }
    KIP_T(4);
}

template <int LOGN, int LOGE, int LOGNB, int NTR, int NDIG>
static hks_status go_kip(FusedKipArgs &a, cudaStream_t s) {
    constexpr int threads = NTR * ((1 << LOGNB) << (LOGN - LOGE));
    constexpr size_t smem = (size_t)NTR * ((1 << LOGN) + ((1 << LOGN) >> LOGE)) * (1 << LOGNB) * sizeof(u64) +
                            (HKS_KIP_TMA ? (size_t)2 * NDIG * (1 << LOGN) * (1 << LOGNB) * sizeof(u64) : 0) +
                            (HKS_KIP_TWS ? (size_t)(1 << LOGN) * (1 << LOGNB) * sizeof(ulonglong2) : 0);
    auto kern = k_ntt_kip<LOGN, LOGE, LOGNB, NTR, NDIG>;
    if (smem > 48 * 1024) {
        hks_func_smem((const void *)kern, smem);
    }
    a.tiles = (1u << a.log_r) >> LOGNB;
    ProfScope ps(K_NTT_ROWS_KIP, s);
    (void)hks_launch_ex(pdl_enabled(), t_win, kern, dim3(a.nu * a.tiles), dim3(threads), smem, s, a);
    HKS_CHECK_LAUNCH();
    // algorithmic words: D read once (pass-1 output or c1), key 2 limbs per (u, j), acc 2 limbs per u
    const double nn = (double)(1ull << a.log_n);
    double nntt = 0;
    for (u32 u = 0; u < a.nu; u++) nntt += a.map.ntr[u];
    const double ndirect = (double)a.nu * NDIG - nntt;
    double ny = 0;
    for (u32 u = 0; u < a.nu; u++) ny += (a.y && a.map.yslot[u] != 0xffff) ? 2.0 : 0.0;
    const double muls = (nntt + ny) * (nn / 2.0) * a.log_c * 7.0 + (double)a.nu * NDIG * 2.0 * nn * 4.0;
    ps.done((nntt + ndirect + 2.0 * a.nu * NDIG + 2.0 * a.nu) * nn * 8.0, muls);
    return HKS_OK;
}

template <int LOGN, int LOGE, int LOGNB>
static hks_status go_kip_d(FusedKipArgs &a, cudaStream_t s) {
#define KC(T, D) if (a.ntr == T && a.ndig == D) return go_kip<LOGN, LOGE, LOGNB, T, D>(a, s);
    KC(1, 1) KC(2, 1) KC(1, 2) KC(2, 2) KC(2, 3) KC(3, 3) KC(3, 4) KC(4, 4)
#if HKS_KIP_XWARP
    KC(4, 3)
#endif
#undef KC
    if (a.ntr == 0) { a.ntr = 1; return go_kip_d<LOGN, LOGE, LOGNB>(a, s); }   // all-direct launch
    HKS_FAIL(HKS_EINVAL, "ntt_kip: %u transformed of %u digits", a.ntr, a.ndig);
}

#ifndef HKS_KIP_KARA
#define HKS_KIP_KARA 1    // Karatsuba products in the key inner product of the fused row pass
#endif
#ifndef HKS_KIP_LOGE
#define HKS_KIP_LOGE 4    // radix-2^LOGE rounds of the fused row pass at log N = 16
#endif
#ifndef HKS_KIP_LOGNB
#define HKS_KIP_LOGNB 1   // 2 rows per CTA: many small CTAs keep the three phases of co-resident CTAs staggered
#endif                    // (measured: 4 rows 98.7 us, 2 rows 96.5 us per C2 KeySwitch)
#ifndef HKS_KIP_LOGNB16
#define HKS_KIP_LOGNB16 2 // at N = 2^16, with per-warp row barriers: 4 rows per CTA (the same 86.3 us per launch alone,
#endif                    // C2 4 938 -> 4 984 KS/s with three concurrent KeySwitches; at N = 2^17 slower: 2 rows kept)
hks_status launch_ntt_kip(const hks_ctx *ctx, FusedKipArgs &a, cudaStream_t s) {
    t_win = &ctx->tw_win;
    a.log_n = ctx->log_n;
    a.log_r = ctx->log_r;
    a.log_c = ctx->log_c;
    if (a.ndig > FK_MAXD || a.nu > FK_MAXU || a.ntr > (a.ndig > 2 ? a.ndig + HKS_KIP_XWARP : 2))
        HKS_FAIL(HKS_EINVAL, "ntt_kip: %u digits (%u transformed) / %u limbs per launch", a.ndig, a.ntr, a.nu);
    switch (ctx->log_n) {
        case 17: return go_kip_d<8, 4, HKS_KIP_LOGNB>(a, s);
        case 16: return go_kip_d<8, HKS_KIP_LOGE, HKS_KIP_LOGNB16>(a, s);
        case 15: return go_kip_d<7, 4, 3>(a, s);
        case 14: return go_kip_d<7, 4, 3>(a, s);
        case 13: return go_kip_d<6, 3, 3>(a, s);
        case 12: return go_kip_d<6, 3, 3>(a, s);
        case 11: return go_kip_d<5, 3, 3>(a, s);
        case 10: return go_kip_d<5, 3, 3>(a, s);
        default: break;
    }
    HKS_FAIL(HKS_EINVAL, "ntt_kip: unsupported log_n %u", ctx->log_n);
}

hks_status run_ntt_kip(const hks_ctx *ctx, const std::vector<KipItem> &items_in, u32 ndig, const u64 *ext,
                       const u64 *c1, const u64 *evk, u64 *acc, u32 nkey, u32 acc_stride, cudaStream_t s,
                       u64 *y, u32 ystride) {
    // heaviest limbs first (more transformed terms; special limbs also run ModDown's inverse row pass), so
    // the grid's tail is made of light CTAs (measured at C2: the special limbs last formed a ~20 us tail)
    std::vector<KipItem> items(items_in);
    auto weight = [&](const KipItem &it) {
        u32 w = (y && it.yslot != 0xffff) ? 2 : 0;
        for (u32 j = 0; j < ndig; j++) w += (it.src[j] & FK_DIRECT) ? 0 : 1;
        return w;
    };
    std::stable_sort(items.begin(), items.end(),
                     [&](const KipItem &a, const KipItem &b) { return weight(a) > weight(b); });
    for (size_t u0 = 0; u0 < items.size(); u0 += FK_MAXU) {
        FusedKipArgs a{};
        a.ext = ext;
        a.c1 = c1;
        a.evk = evk;
        a.acc = acc;
        a.pc = ctx->d_pc;
        a.tw = ctx->d_tw_row_fwd;
        a.nu = (u32)std::min<size_t>(FK_MAXU, items.size() - u0);
        a.ndig = ndig;
        a.ntr = 0;
        a.nkey = nkey;
        a.acc_stride = acc_stride;
        a.y = y;
        a.ystride = ystride;
        a.tw_inv = ctx->d_tw_row_inv;
        for (u32 uu = 0; uu < a.nu; uu++) {
            const KipItem &it = items[u0 + uu];
            a.map.prime[uu] = it.prime;
            a.map.kslot[uu] = it.kslot;
            a.map.aslot[uu] = it.aslot;
            a.map.yslot[uu] = y ? it.yslot : (u16)0xffff;
            u32 i = 0, ntr = 0;
            for (u32 pass = 0; pass < 2; pass++)          // transformed terms first, then direct
                for (u32 j = 0; j < ndig; j++) {
                    const bool direct = (it.src[j] & FK_DIRECT) != 0;
                    if (direct != (pass == 1)) continue;
                    a.map.dsrc[uu][i] = it.src[j];
                    a.map.dig[uu][i] = (u8)j;
                    i++;
                    ntr += direct ? 0 : 1;
                }
            a.map.ntr[uu] = (u8)ntr;
            a.ntr = std::max(a.ntr, ntr);
        }
        // ModDown's inverse row pass (y mode) needs two thread groups, one per accumulator
        bool anyy = false;
        for (u32 uu = 0; uu < a.nu; uu++) anyy |= a.map.yslot[uu] != 0xffff;
        if (anyy && a.ntr < 2) a.ntr = 2;
#if HKS_KIP_XWARP
        if (a.ntr == 3 && ndig == 3) a.ntr = 4;   // a fourth warp: idle in the row pass, 2 product steps per thread
#endif
        hks_status st = launch_ntt_kip(ctx, a, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}
