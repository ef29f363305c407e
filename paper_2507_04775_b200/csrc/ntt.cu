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
#include "internal.h"

template <int LOGN, int LOGE, int LOGNB, bool COLS, bool FWD, int EPI>
__global__ void __launch_bounds__((1 << LOGNB) << (LOGN - LOGE))
k_ntt(const __grid_constant__ NttArgs A) {
    constexpr int n = 1 << LOGN;
    constexpr int E = 1 << LOGE;
    constexpr int NB = 1 << LOGNB;
    constexpr int TPS = n >> LOGE;                    // threads per sub-transform
    constexpr int NR = (LOGN + LOGE - 1) / LOGE;      // rounds
    constexpr int ROWPAD = n + (n >> LOGE);
    extern __shared__ __align__(16) u64 sm[];

    const u32 b = blockIdx.x / A.tiles;
    const u32 tile = blockIdx.x - b * A.tiles;
    const u32 prime = A.map.prime[b];
    const u32 log_n = A.log_n;
    const size_t N = (size_t)1 << log_n;
    const u64 *__restrict__ src = A.in + (size_t)A.map.sin[b] * N;
    u64 *__restrict__ dst = A.out + (size_t)A.map.sout[b] * N;
    const u64 p = A.pc[prime].p;
    const u64 two_p = 2 * p;
    const u32 C = 1u << A.log_c;
    const int tid = threadIdx.x;
    const int bsub = COLS ? (tid & (NB - 1)) : (tid >> (LOGN - LOGE));
    const int tu = COLS ? (tid >> LOGNB) : (tid & (TPS - 1));
    const u32 gcol = COLS ? tile * NB + bsub : 0;
    const u32 grow = COLS ? 0 : tile * NB + bsub;
    const ulonglong2 *__restrict__ tw =
        COLS ? A.tw + (size_t)prime * n : A.tw + (((size_t)prime << A.log_r) + grow) * n;

    auto gidx = [&](int k) -> size_t { return COLS ? (size_t)k * C + gcol : (size_t)grow * C + k; };
    auto saddr = [&](int k) -> int {
        return COLS ? (k + (k >> LOGE)) * NB + bsub : bsub * ROWPAD + k + (k >> LOGE);
    };

    // epilogue constants
    ulonglong2 sc = make_ulonglong2(0, 0);
    if (EPI == EPI_SCALE) sc = A.scale ? A.scale[b % A.scale_mod] : A.ninv[prime];
    ulonglong2 pinv = make_ulonglong2(0, 0);
    const u64 *ea = nullptr, *eb = nullptr;
    if (EPI == EPI_MODDOWN) {
        pinv = A.pinv[prime];
        ea = A.ea + (size_t)A.map.sa[b] * N;
        eb = (A.eb && A.map.sb[b] != 0xffff) ? A.eb + (size_t)A.map.sb[b] * N : nullptr;
    }
    auto epi = [&](u64 x, int k) -> u64 {
        if (EPI == EPI_LAZY) return x;
        if (EPI == EPI_SCALE) return shoup(x, sc.x, sc.y, p);
        u64 y = csub(csub(x, two_p), p);
        if (EPI == EPI_CANON) return y;
        // EPI_MODDOWN: (a - y) * P^-1 [+ b]
        const size_t xg = gidx(k);
        u64 r = shoup(ea[xg] + p - y, pinv.x, pinv.y, p);
        if (eb) {
            const size_t xs = A.galois == 1 ? xg : (size_t)automorph_src((u32)xg, log_n, A.galois);
            r = csub(r + eb[xs], p);
        }
        return r;
    };

    // inverse ROWS (first inverse pass) reads the tile through shared memory: per-thread elements
    // of its first round are contiguous, so a direct load would not coalesce.
    if (!FWD && !COLS) {
        for (int idx = tid; idx < NB * n; idx += NB * TPS) {
            const int r = idx >> LOGN, k = idx & (n - 1);
            sm[r * ROWPAD + k + (k >> LOGE)] = src[(size_t)(tile * NB + r) * C + k];
        }
        __syncthreads();
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
        if (rr > 0) __syncthreads();

        // gather
#pragma unroll
        for (int q = 0; q < UPT; q++) {
            const int uid = tu * UPT + q;
            const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
            for (int k = 0; k < Ee; k++) {
                const int j = base + (k << lstride);
                v[q * Ee + k] = from_global ? src[gidx(j)] : sm[saddr(j)];
            }
        }
        // butterflies
#pragma unroll
        for (int q = 0; q < UPT; q++) {
            const int uid = tu * UPT + q;
            const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
            for (int l = 0; l < e; l++) {
                const int lt = FWD ? (e - 1 - l) : l;
                const int t = 1 << lt;
                const int ltg = lt + lstride;
#pragma unroll
                for (int k = 0; k < Ee; k++) {
                    if (k & t) continue;
                    const int j = base + (k << lstride);
                    const ulonglong2 w = __ldg(&tw[(n + j) >> (ltg + 1)]);
                    if (FWD)
                        ct_bfly(v[q * Ee + k], v[q * Ee + k + t], w.x, w.y, p, two_p);
                    else
                        gs_bfly(v[q * Ee + k], v[q * Ee + k + t], w.x, w.y, p, two_p);
                }
            }
        }
        // scatter
        const bool via_smem_out = last && FWD && !COLS;
        if (!last || via_smem_out) {
            if (rr > 0 || !from_global) __syncthreads();
#pragma unroll
            for (int q = 0; q < UPT; q++) {
                const int uid = tu * UPT + q;
                const int base = ((uid >> lstride) << lBsz) + (uid & ((1 << lstride) - 1));
#pragma unroll
                for (int k = 0; k < Ee; k++) {
                    const int j = base + (k << lstride);
                    sm[saddr(j)] = last ? epi(v[q * Ee + k], j) : v[q * Ee + k];
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
                    dst[gidx(j)] = epi(v[q * Ee + k], j);
                }
            }
        }
    }
    if (FWD && !COLS) {
        __syncthreads();
        for (int idx = tid; idx < NB * n; idx += NB * TPS) {
            const int r = idx >> LOGN, k = idx & (n - 1);
            dst[(size_t)(tile * NB + r) * C + k] = sm[r * ROWPAD + k + (k >> LOGE)];
        }
    }
}

template <int LOGN, int LOGE, int LOGNB, bool COLS, bool FWD, int EPI>
static hks_status go(NttArgs &a, cudaStream_t s) {
    constexpr int threads = (1 << LOGNB) << (LOGN - LOGE);
    constexpr size_t smem = (size_t)((1 << LOGN) + ((1 << LOGN) >> LOGE)) * (1 << LOGNB) * sizeof(u64);
    auto kern = k_ntt<LOGN, LOGE, LOGNB, COLS, FWD, EPI>;
    if (smem > 48 * 1024) {
        static bool once = [&] {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            return true;
        }();
        (void)once;
    }
    a.tiles = COLS ? ((1u << a.log_c) >> LOGNB) : ((1u << a.log_r) >> LOGNB);
    const int cls = FWD ? (COLS ? K_NTT_FWD_COLS : (EPI == EPI_MODDOWN ? K_NTT_FWD_ROWS_MODDOWN : K_NTT_FWD_ROWS))
                        : (COLS ? K_NTT_INV_COLS : K_NTT_INV_ROWS);
    ProfScope ps(cls, s);
    kern<<<a.nlimbs * a.tiles, threads, smem, s>>>(a);
    HKS_CHECK_LAUNCH();
    // algorithmic bytes: each limb read once and written once (+ ModDown operands acc, c0)
    double words = 2.0 * a.nlimbs;
    if (EPI == EPI_MODDOWN) words += a.nlimbs * (a.eb ? 2.0 : 1.0);
    ps.done(words * (double)(1ull << a.log_n) * 8.0);
    return HKS_OK;
}

// per ring size: sub-transform shapes for the column pass (length R) and the row pass (length C)
#define NTT_SHAPES(X)                  \
    X(17, 9, 4, 3, 8, 4, 4)            \
    X(16, 8, 4, 4, 8, 4, 4)            \
    X(15, 8, 4, 4, 7, 4, 4)            \
    X(14, 7, 4, 4, 7, 4, 4)            \
    X(13, 7, 4, 4, 6, 3, 4)            \
    X(12, 6, 3, 4, 6, 3, 4)            \
    X(11, 6, 3, 4, 5, 3, 4)            \
    X(10, 5, 3, 4, 5, 3, 4)

hks_status launch_ntt_pass(const hks_ctx *ctx, NttDir dir, int pass, int epi, NttArgs &a, cudaStream_t s) {
    a.log_n = ctx->log_n;
    a.log_r = ctx->log_r;
    a.log_c = ctx->log_c;
    const bool cols = (dir == NTT_FWD) ? (pass == 0) : (pass == 1);
    switch (ctx->log_n) {
#define X(LN, LR, ER, BR, LC, EC, BC)                                                               \
    case LN:                                                                                        \
        if (dir == NTT_FWD && cols) return go<LR, ER, BR, true, true, EPI_LAZY>(a, s);              \
        if (dir == NTT_FWD && epi == EPI_CANON) return go<LC, EC, BC, false, true, EPI_CANON>(a, s); \
        if (dir == NTT_FWD && epi == EPI_MODDOWN)                                                   \
            return go<LC, EC, BC, false, true, EPI_MODDOWN>(a, s);                                  \
        if (dir == NTT_INV && !cols) return go<LC, EC, BC, false, false, EPI_LAZY>(a, s);           \
        if (dir == NTT_INV && cols) return go<LR, ER, BR, true, false, EPI_SCALE>(a, s);            \
        break;
        NTT_SHAPES(X)
#undef X
        default:
            break;
    }
    HKS_FAIL(HKS_EINVAL, "ntt: unsupported log_n %u / epilogue %d", ctx->log_n, epi);
}

static void fill_map(NttArgs &a, const LimbList &L, size_t off, u32 cnt, bool second_pass) {
    for (u32 i = 0; i < cnt; i++) {
        a.map.sin[i] = second_pass ? L.sout[off + i] : L.sin[off + i];
        a.map.sout[i] = L.sout[off + i];
        a.map.prime[i] = L.prime[off + i];
        a.map.sa[i] = L.sa[off + i];
        a.map.sb[i] = L.sb[off + i];
    }
    a.nlimbs = cnt;
}

hks_status run_ntt(const hks_ctx *ctx, NttDir dir, const LimbList &L, const u64 *in, u64 *out,
                   const ulonglong2 *scale, u32 scale_mod, cudaStream_t s) {
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
        a.tw = dir == NTT_FWD ? ctx->d_tw_col_fwd : ctx->d_tw_row_inv;
        hks_status st = launch_ntt_pass(ctx, dir, 0, EPI_LAZY, a, s);
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

hks_status run_ntt_moddown(const hks_ctx *ctx, const LimbList &L, u64 *buf, u64 *out, const u64 *acc,
                           const u64 *c0, u64 galois, cudaStream_t s) {
    for (size_t off = 0; off < L.size(); off += HKS_MAXB) {
        u32 cnt = (u32)((L.size() - off) < HKS_MAXB ? (L.size() - off) : HKS_MAXB);
        NttArgs a{};
        a.pc = ctx->d_pc;
        a.ninv = ctx->d_ninv;
        a.pinv = ctx->d_pinv;
        a.galois = galois;
        // pass 0: columns, in place on buf (slots sin)
        for (u32 i = 0; i < cnt; i++) {
            a.map.sin[i] = L.sin[off + i];
            a.map.sout[i] = L.sin[off + i];
            a.map.prime[i] = L.prime[off + i];
        }
        a.nlimbs = cnt;
        a.in = buf;
        a.out = buf;
        a.tw = ctx->d_tw_col_fwd;
        hks_status st = launch_ntt_pass(ctx, NTT_FWD, 0, EPI_LAZY, a, s);
        if (st != HKS_OK) return st;
        // pass 1: rows, buf -> out with the ModDown epilogue
        fill_map(a, L, off, cnt, false);
        a.in = buf;
        a.out = out;
        a.ea = acc;
        a.eb = c0;
        a.tw = ctx->d_tw_row_fwd;
        st = launch_ntt_pass(ctx, NTT_FWD, 1, EPI_MODDOWN, a, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}
