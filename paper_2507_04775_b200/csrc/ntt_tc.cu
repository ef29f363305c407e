// ntt_tc.cu -- the column pass of the N = 2^16 NTT on the tcgen05 tensor cores.
//
// The column pass (8 butterfly stages on each 256-row column, §3.6.4) is exactly two
// rounds of 16-point transforms with a diagonal twist between them (ctx.cu builds the tables):
//   forward:  y = W_B[0] · diag(twist) · W_A   (round 1 on the stride-16 classes {v + 16k}, round 2 on
//             the 16-row blocks {16v + k})
//   inverse:  y = W'_A · diag(twist) · W'_B[0] (round 1 on the blocks, round 2 on the classes), then the
//             EPI_SCALE factor and a canonical store.
// Each round multiplies 16-word vectors by a 16 x 16 matrix mod p with the byte-split identity of
// k_bconv_tc: A = the vectors' bytes (K = 128), B = the matrix image (N = 16 outputs x 8 byte columns),
// D in TMEM, one tcgen05.ld + 14-instruction reduction per output.  Per element that is two reductions
// and one Shoup product (the twist) instead of the eight butterfly half-products of the butterfly pass:
// ~48 instead of ~112 FMA-heavy-pipe cycles per warp and 32 elements.
//
// A tile = (limb, 8 columns): 128 vectors per round = one M = 128 MMA of K = 128 (four k32 steps).  The
// kernel is persistent (one CTA per SM, contiguous balanced tile ranges, so a CTA meets one or two limbs)
// and warp-specialised, every hand-off an mbarrier:
//   warps 0-2   loaders: cp.async of the next tiles' round-1 operands (8-byte elements, transposed into
//               the K-major A layout) into S1 stages, plus the B images of each new prime into one of two
//               table slots;
//   warp 3      one thread issues the MMAs: round 1 of tile j, then round 2 of tile j - 1, each into its
//               own double-buffered TMEM accumulator (4 x 128 of the 512 columns);
//   warps 4-11  round-1 epilogue: TMEM -> reduce -> twist -> round 2's A operand in shared memory;
//   warps 12-19 round-2 epilogue: TMEM -> reduce (-> scale) -> global stores.
// Outputs are congruent to the butterfly pass's: forward lazily reduced to [0, 3p) (the row pass accepts
// [0, 8p + 2^32)), inverse scaled and canonical.
#include <algorithm>

#include "internal.h"
#include "tc.cuh"

#define NC_CW 8                 // columns per tile
#define NC_TPL (256 / NC_CW)    // tiles per limb
#ifndef NC_S1
#define NC_S1 4                 // round-1 operand stages
#endif
#define NC_S2 2                 // round-2 operand stages
#define NC_LOADW 3              // loader warps
#define NC_E1W 8                // round-1 epilogue warps
#define NC_E2W 8                // round-2 epilogue warps
#define NC_THREADS ((NC_LOADW + 1 + NC_E1W + NC_E2W) * 32)
#define NC_OPB 16384            // bytes of one operand stage (128 vectors x 128 bytes)
#define NC_TABB 32768           // bytes of one table slot (round-1 and round-2 images)
#define NC_SMEM (NC_S1 * NC_OPB + NC_S2 * NC_OPB + 2 * NC_TABB)

struct NttColsArgs {
    const u64 *in;
    u64 *out;
    const u64 *tab;             // [prime][NTT16_TAB]: round-1 image, round-2 image, twist (w, w')[16][16]
    const ulonglong2 *scale;    // inverse: scale[b % scale_mod] or, if NULL, ninv[prime]
    const ulonglong2 *ninv;
    const PrimeConst *pc;
    u32 nlimbs, scale_mod;
    LimbMap map;
};

__device__ __forceinline__ void cp_async16(u32 saddr, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <bool FWD>
__global__ void __launch_bounds__(NC_THREADS, 1) k_ntt_cols_tc(const __grid_constant__ NttColsArgs A) {
    pdl_trigger();
    constexpr u32 N = 1u << 16;
    extern __shared__ __align__(1024) uint8_t csm[];
    __shared__ __align__(8) u64 a1_full[NC_S1], a1_empty[NC_S1], a2_full[NC_S2], a2_empty[NC_S2];
    __shared__ __align__(8) u64 mma1_done[2], mma2_done[2], t1_empty[2], t2_empty[2], slot_free[2];
    __shared__ u32 tmem_s;
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const u32 ntile = A.nlimbs * NC_TPL;
    const u32 t_beg = (u32)((u64)blockIdx.x * ntile / gridDim.x);      // balanced contiguous ranges
    const u32 t_end = (u32)((u64)(blockIdx.x + 1) * ntile / gridDim.x);
    const u32 nloc = t_end - t_beg;
    const u32 b_first = t_beg / NC_TPL;
    // table segment of local tile j: the limb offset from the CTA's first limb (slot = segment & 1)
    auto seg = [&](u32 j) { return (t_beg + j) / NC_TPL - b_first; };
    auto last_of_seg = [&](u32 j) { return j + 1 == nloc || seg(j + 1) != seg(j); };

    if (tid == 0) {
        for (int s = 0; s < NC_S1; s++) {
            mbar_init(smem_u32(&a1_full[s]), NC_LOADW * 32);
            mbar_init(smem_u32(&a1_empty[s]), 1);
        }
        for (int s = 0; s < NC_S2; s++) {
            mbar_init(smem_u32(&a2_full[s]), NC_E1W);
            mbar_init(smem_u32(&a2_empty[s]), 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(smem_u32(&mma1_done[b]), 1);
            mbar_init(smem_u32(&mma2_done[b]), 1);
            mbar_init(smem_u32(&t1_empty[b]), NC_E1W);
            mbar_init(smem_u32(&t2_empty[b]), NC_E2W);
            mbar_init(smem_u32(&slot_free[b]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 3) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const u32 tmem = tmem_s;
    pdl_wait();

    const u32 op1 = smem_u32(csm), op2 = op1 + NC_S1 * NC_OPB, tab0 = op2 + NC_S2 * NC_OPB;
    // element k of round-1 / round-2 vector class v sits in row row1(v, k) / row2(v, k) of the column
    auto row1 = [](u32 v, u32 k) { return FWD ? v + 16 * k : 16 * v + k; };
    auto row2 = [](u32 v, u32 k) { return FWD ? 16 * v + k : v + 16 * k; };

    if (warp < NC_LOADW) {
        // ---------------- loaders ----------------
        const u32 lt = tid;   // 0 .. 95
        auto arrive_full = [&](u32 j) {
            fence_async_smem();
            mbar_arrive(smem_u32(&a1_full[j % NC_S1]));
        };
        constexpr u32 LAG = NC_S1 - 1;   // tiles whose copies may be in flight unsignalled
        u32 na = 0;                      // next tile whose a1_full arrival is due
        for (u32 j = 0; j < nloc; j++) {
            const u32 s = j % NC_S1;
            if (j >= NC_S1) mbar_wait(smem_u32(&a1_empty[s]), ((j / NC_S1) - 1) & 1);
            const u32 tile = t_beg + j, b = tile / NC_TPL, c0 = (tile % NC_TPL) * NC_CW;
            if (j == 0 || seg(j) != seg(j - 1)) {
                // a new limb: its prime's round-1 / round-2 images into table slot seg & 1, after the last
                // round-2 MMA of segment seg - 2 released it -- which needs every earlier tile signalled first
                const u32 k = seg(j);
                if (k >= 2) {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                    while (na < j) arrive_full(na++);
                    mbar_wait(smem_u32(&slot_free[k & 1]), ((k - 2) >> 1) & 1);
                }
                const uint8_t *t = reinterpret_cast<const uint8_t *>(A.tab + (size_t)A.map.prime[b] * NTT16_TAB);
                const u32 dst = tab0 + (k & 1) * NC_TABB;
                for (u32 o = lt * 16; o < NC_TABB; o += NC_LOADW * 32 * 16) cp_async16(dst + o, t + o);
            }
            // element (vector m = v * 8 + c, k): row row1(v, k), column c0 + c -> A layout
            const u64 *src = A.in + (size_t)A.map.sin[b] * N + c0;
            const u32 base = op1 + s * NC_OPB;
            for (u32 e = lt; e < 2048; e += NC_LOADW * 32) {
                const u32 c = e & 7, v = (e >> 3) & 15, k = e >> 7;
                cp_async8(base + v * 1024 + (k >> 1) * 128 + c * 16 + (k & 1) * 8, src + (size_t)row1(v, k) * 256 + c);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            if (j + 1 - na > LAG) {          // groups na .. j pending: complete the oldest
                asm volatile("cp.async.wait_group %0;" ::"n"(LAG) : "memory");
                arrive_full(na++);
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        while (na < nloc) arrive_full(na++);
    } else if (warp == NC_LOADW) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const u32 idesc = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);   // M = N = 128, s32 += u8 x u8
            auto round2 = [&](u32 i) {
                const u32 s = i % NC_S2;
                mbar_wait(smem_u32(&a2_full[s]), (i / NC_S2) & 1);
                if (i >= 2) mbar_wait(smem_u32(&t2_empty[i & 1]), ((i >> 1) - 1) & 1);
                tc_fence_after();
                fence_async_smem();
                const u32 a = op2 + s * NC_OPB, bimg = tab0 + (seg(i) & 1) * NC_TABB + NC_TABB / 2;
#pragma unroll
                for (int k = 0; k < 4; k++)
                    tc_mma_i8(tmem + 256 + (i & 1) * 128, tc_desc(a + k * 256, 128, 1024), tc_desc(bimg + k * 256, 128, 1024),
                              idesc, k > 0 ? 1u : 0u);
                tc_commit(smem_u32(&a2_empty[s]));
                tc_commit(smem_u32(&mma2_done[i & 1]));
                if (last_of_seg(i)) tc_commit(smem_u32(&slot_free[seg(i) & 1]));
            };
            for (u32 j = 0; j < nloc; j++) {
                const u32 s = j % NC_S1;
                mbar_wait(smem_u32(&a1_full[s]), (j / NC_S1) & 1);
                if (j >= 2) mbar_wait(smem_u32(&t1_empty[j & 1]), ((j >> 1) - 1) & 1);
                tc_fence_after();
                fence_async_smem();
                const u32 a = op1 + s * NC_OPB, bimg = tab0 + (seg(j) & 1) * NC_TABB;
#pragma unroll
                for (int k = 0; k < 4; k++)
                    tc_mma_i8(tmem + (j & 1) * 128, tc_desc(a + k * 256, 128, 1024), tc_desc(bimg + k * 256, 128, 1024),
                              idesc, k > 0 ? 1u : 0u);
                tc_commit(smem_u32(&a1_empty[s]));
                tc_commit(smem_u32(&mma1_done[j & 1]));
                if (j >= 1) round2(j - 1);
            }
            if (nloc) round2(nloc - 1);
        }
        __syncwarp();
    } else if (warp < NC_LOADW + 1 + NC_E1W) {
        // ---------------- round-1 epilogue: reduce, twist, round 2's operand ----------------
        const u32 ew = warp - (NC_LOADW + 1);
        const u32 q = warp & 3, half = ew >> 2;            // TMEM lane quarter; outputs [8 half, 8 half + 8)
        const u32 m = q * 32 + lane, v = m >> 3, c = m & 7;  // this lane's vector (class / block v, column c)
        for (u32 j = 0; j < nloc; j++) {
            const u32 tile = t_beg + j, b = tile / NC_TPL;
            const PrimeConst pc = A.pc[A.map.prime[b]];
            const u64 np = 0 - pc.p;
            const u32 mu = (u32)pc.mu80;
            const ulonglong2 *tw = reinterpret_cast<const ulonglong2 *>(A.tab + (size_t)A.map.prime[b] * NTT16_TAB + 2 * NTT16_IMG) + v * 16;
            mbar_wait(smem_u32(&mma1_done[j & 1]), (j >> 1) & 1);
            tc_fence_after();
            const u32 s2 = j % NC_S2;
            if (j >= NC_S2) mbar_wait(smem_u32(&a2_empty[s2]), ((j / NC_S2) - 1) & 1);
            const u32 tb = tmem + (j & 1) * 128 + ((q * 32) << 16);
            // round-2 vector o * 8 + c, element v
            const u32 w2 = op2 + s2 * NC_OPB + (v >> 1) * 128 + c * 16 + (v & 1) * 8;
#pragma unroll
            for (u32 o0 = 0; o0 < 8; o0 += 4) {
                u32 r[4][8];
#pragma unroll
                for (int k = 0; k < 4; k++) tc_ld8(tb + (8 * half + o0 + k) * 8, r[k]);
                tc_wait_ld();
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const u32 o = 8 * half + o0 + k;
                    const u64 x = bytesum_reduce_c<true>(r[k], np, mu);   // [0, 3p)
                    const ulonglong2 t = __ldg(tw + o);
                    const u64 y = shoup_approx(x, t.x, t.y, np);          // [0, 4p)
                    asm volatile("st.shared.u64 [%0], %1;" ::"r"(w2 + o * 1024), "l"(y) : "memory");
                }
            }
            fence_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(smem_u32(&t1_empty[j & 1]));
                mbar_arrive(smem_u32(&a2_full[s2]));
            }
        }
    } else {
        // ---------------- round-2 epilogue: reduce (scale), store ----------------
        const u32 ew = warp - (NC_LOADW + 1 + NC_E1W);
        const u32 q = warp & 3, half = ew >> 2;
        const u32 m = q * 32 + lane, g = m >> 3, c = m & 7;
        for (u32 j = 0; j < nloc; j++) {
            const u32 tile = t_beg + j, b = tile / NC_TPL, c0 = (tile % NC_TPL) * NC_CW;
            const u32 prime = A.map.prime[b];
            const PrimeConst pc = A.pc[prime];
            const u64 np = 0 - pc.p;
            const u32 mu = (u32)pc.mu80;
            ulonglong2 sc = make_ulonglong2(0, 0);
            if (!FWD) sc = A.scale ? A.scale[b % A.scale_mod] : A.ninv[prime];
            u64 *dst = A.out + (size_t)A.map.sout[b] * N + c0 + c;
            mbar_wait(smem_u32(&mma2_done[j & 1]), (j >> 1) & 1);
            tc_fence_after();
            const u32 tb = tmem + 256 + (j & 1) * 128 + ((q * 32) << 16);
#pragma unroll
            for (u32 o0 = 0; o0 < 8; o0 += 4) {
                u32 r[4][8];
#pragma unroll
                for (int k = 0; k < 4; k++) tc_ld8(tb + (8 * half + o0 + k) * 8, r[k]);
                tc_wait_ld();
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const u32 o = 8 * half + o0 + k;
                    u64 x = bytesum_reduce_c<true>(r[k], np, mu);
                    if (!FWD) x = csub(csub(shoup_approx(x, sc.x, sc.y, np), 2 * pc.p), pc.p);
                    dst[(size_t)row2(g, o) * 256] = x;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&t2_empty[j & 1]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

hks_status launch_ntt_cols_tc(const hks_ctx *ctx, NttDir dir, int /*epi*/, const NttArgs &na, cudaStream_t s) {
    constexpr size_t smem = NC_SMEM;
    const int nsm = hks_num_sms();
    hks_func_smem((const void *)k_ntt_cols_tc<true>, smem);
    hks_func_smem((const void *)k_ntt_cols_tc<false>, smem);
    NttColsArgs a;
    a.in = na.in;
    a.out = na.out;
    a.tab = dir == NTT_FWD ? ctx->d_ntt_img_fwd : ctx->d_ntt_img_inv;
    a.scale = na.scale;
    a.ninv = ctx->d_ninv;
    a.pc = ctx->d_pc;
    a.nlimbs = na.nlimbs;
    a.scale_mod = na.scale_mod ? na.scale_mod : 1;
    a.map = na.map;
    const u32 grid = std::min<u32>(a.nlimbs * NC_TPL, (u32)nsm);
    ProfScope ps(dir == NTT_FWD ? K_NTT_FWD_COLS : K_NTT_INV_COLS, s);
    const cudaError_t e = dir == NTT_FWD
                              ? hks_launch(k_ntt_cols_tc<true>, dim3(grid), dim3(NC_THREADS), smem, s, a)
                              : hks_launch(k_ntt_cols_tc<false>, dim3(grid), dim3(NC_THREADS), smem, s, a);
    const double nn = 65536.0;
    // algorithmic work: the butterflies the pass replaces are not counted as integer-pipe products (they run
    // as tensor-core MMAs); the twist and, for the inverse, the scale are one Shoup product per element each
    ps.done(2.0 * a.nlimbs * nn * 8.0, a.nlimbs * nn * 7.0 * (dir == NTT_FWD ? 1.0 : 2.0));
    if (e != cudaSuccess) HKS_FAIL(HKS_ECUDA, "k_ntt_cols_tc launch: %s", cudaGetErrorString(e));
    return HKS_OK;
}
