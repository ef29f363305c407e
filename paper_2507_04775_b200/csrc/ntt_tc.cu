// ntt_tc.cu -- the column pass of the N = 2^16 NTT on the tcgen05 tensor cores (opt-in, HKS_NTT_TC=1;
// DESIGN.md §5).
//
// The column pass (8 butterfly stages on each 256-row column, §3.6.4) is exactly two
// rounds of 16-point transforms with a diagonal twist between them (ctx.cu builds the tables):
//   forward:  y = W_B[0] · diag(twist) · W_A   (round 1 on the stride-16 classes {v + 16k}, round 2 on
//             the 16-row blocks {16v + k})
//   inverse:  y = W'_A · diag(twist) · W'_B[0] (round 1 on the blocks, round 2 on the classes), then the
//             EPI_SCALE factor and a canonical store.
// Each round multiplies 16-word vectors by a 16 x 16 matrix mod p with the byte-split identity of
// k_bconv_tc: A = the vectors' bytes (K = 128), B = the matrix image (N = 16 outputs x 8 byte columns),
// D in TMEM, one tcgen05.ld + 14-instruction reduction per output.  A CTA owns a (limb, 32-column) tile
// (256 rows x 32 columns, 64 KB) that stays in shared memory between the rounds: round-1 outputs are
// twisted (one Shoup product) and written straight into round 2's operand layout, over the round-1
// operands already consumed.  Outputs are congruent to the butterfly pass's, lazily reduced to [0, 4p),
// except the inverse pass, which is scaled and canonical.
#include <algorithm>

#include "internal.h"
#include "tc.cuh"

#if HKS_EXPERIMENTAL

#ifndef HKS_NTC_SPLIT
#define HKS_NTC_SPLIT 1   // warps per TMEM lane quarter and M-tile (each takes 16 / SPLIT of the outputs)
#endif
#define NC_THREADS (256 * HKS_NTC_SPLIT)
#define NC_OUT (16 / HKS_NTC_SPLIT)
#define NC_ILP (NC_OUT < 4 ? NC_OUT : 4)

struct NttColsArgs {
    const u64 *in;
    u64 *out;
    const u64 *tab;             // [prime][NTT16_TAB]
    const ulonglong2 *scale;    // inverse: scale[b % scale_mod] or, if NULL, ninv[prime]
    const ulonglong2 *ninv;
    const PrimeConst *pc;
    u32 nlimbs, scale_mod;
    LimbMap map;
};

// Shared memory (dynamic, 1024-aligned): two 32 KB tile buffers (the next tile is loaded into one while
// the current one is processed in the other), [64K, 80K) round-1 image, [80K, 96K) round-2 image,
// [96K, 100K) twist.  A tile = (limb, 16 columns): 256 vectors per round = two 128-row M-tiles, K-major,
// SBO 1024.  Round 1: vector V = (class V / 16, column V % 16); its outputs are twisted into round 2's
// operands in place of the consumed round-1 operands (round-2 vector v2 = output index, element =
// round-1 class).  CTAs take contiguous tile ranges so a CTA rarely changes prime (tables reloaded then).
template <bool FWD>
__global__ void __launch_bounds__(NC_THREADS, 2) k_ntt_cols_tc(const __grid_constant__ NttColsArgs A) {
    pdl_trigger();
    constexpr u32 N = 1u << 16;
    extern __shared__ __align__(1024) uint8_t csm[];
    uint8_t *simg1 = csm + 65536, *simg2 = csm + 81920;
    const ulonglong2 *stw = reinterpret_cast<const ulonglong2 *>(csm + 98304);
    __shared__ __align__(8) u64 mbar;
    __shared__ u32 tmem_s;
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(smem_u32(&mbar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const u32 tmem = tmem_s;
    pdl_wait();

    const u32 idesc = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);   // M = N = 128, s32 += u8 x u8
    const u32 buf_a = smem_u32(csm), img1_a = smem_u32(simg1), img2_a = smem_u32(simg2);
    u32 phase = 0, cur_prime = 0xffffffffu;
    PrimeConst pc{};
    // round-1 / round-2 row of element k of vector class v:  strided v + 16k, blocked 16v + k
    auto row1 = [](u32 v, u32 k) { return FWD ? v + 16 * k : 16 * v + k; };
    auto row2 = [](u32 v, u32 k) { return FWD ? 16 * v + k : v + 16 * k; };
    const u32 ntile = A.nlimbs * 16;
    const u32 t_beg = (u32)((u64)blockIdx.x * ntile / gridDim.x);        // balanced contiguous ranges
    const u32 t_end = (u32)((u64)(blockIdx.x + 1) * ntile / gridDim.x);
    // this thread's two round-1 vectors: V = tid, tid + 256 ... (256 vectors: M-tile V >> 7)
    auto load_tile = [&](u32 tile, u32 buf) {
        const u32 b = tile >> 4, c0 = (tile & 15) * 16;
        const u64 *src = A.in + (size_t)A.map.sin[b] * N + c0;
        const u32 V = tid & 255, mt = V >> 7, m = V & 127, cls = V >> 4, c = V & 15;
        const u32 base = buf_a + buf * 32768 + mt * 16384 + (m >> 3) * 1024 + (m & 7) * 16;
#pragma unroll
        for (int kk = 0; kk < NC_OUT; kk++) {
            const int k = (tid >> 8) * NC_OUT + kk;
            cp_async8(base + (k >> 1) * 128 + (k & 1) * 8, src + (size_t)row1(cls, k) * 256 + c);
        }
    };
    if (t_beg < t_end) load_tile(t_beg, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (u32 tile = t_beg, it = 0; tile < t_end; tile++, it++) {
        const u32 buf = it & 1;
        const u32 b = tile >> 4, c0 = (tile & 15) * 16;
        const u32 prime = A.map.prime[b];
        if (prime != cur_prime) {   // tables of this prime (rare: contiguous tile ranges)
            __syncthreads();
            const uint8_t *t = reinterpret_cast<const uint8_t *>(A.tab + (size_t)prime * NTT16_TAB);
            for (u32 o = tid * 16; o < 36864; o += NC_THREADS * 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(img1_a + o), "l"(t + o) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
            cur_prime = prime;
            pc = A.pc[prime];
        }
        if (tile + 1 < t_end) load_tile(tile + 1, buf ^ 1);   // next tile in flight during this one
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 1;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();

        const u64 np = 0 - pc.p;
        const u32 mu = (u32)pc.mu80;
        const u32 q = warp & 3, mtl = (warp >> 2) & 1, ob = (warp >> 3) * NC_OUT;   // lane quarter, M-tile, outputs
        const u32 sv_a = buf_a + buf * 32768;
        const u32 tb = tmem + mtl * 128 + ((q * 32) << 16);
        // ---- round 1
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int t = 0; t < 2; t++)
#pragma unroll
                for (int s = 0; s < 4; s++)
                    tc_mma_i8(tmem + t * 128, tc_desc(sv_a + t * 16384 + s * 256, 128, 1024),
                              tc_desc(img1_a + s * 256, 128, 1024), idesc, s > 0 ? 1u : 0u);
            tc_commit(smem_u32(&mbar));
        }
        mbar_wait(smem_u32(&mbar), phase);
        phase ^= 1;
        tc_fence_after();
        {
            const u32 m = 32 * q + lane, v1 = 8 * mtl + (m >> 4), c = m & 15;   // this thread's round-1 vector
            // round-2 operand: vector o (M-tile o / 8, row (o % 8) 16 + c), element v1
            const u32 w2 = sv_a + ((c & 8) ? 1024 : 0) + (v1 >> 1) * 128 + (c & 7) * 16 + (v1 & 1) * 8;
#pragma unroll
            for (u32 o0 = ob; o0 < ob + NC_OUT; o0 += NC_ILP) {
                u32 v[NC_ILP][8];
#pragma unroll
                for (int k = 0; k < NC_ILP; k++) tc_ld8(tb + (o0 + k) * 8, v[k]);
                tc_wait_ld();
#pragma unroll
                for (int k = 0; k < NC_ILP; k++) {
                    const u32 o = o0 + k;
                    const u64 r = bytesum_reduce_c<true>(v[k], np, mu);   // [0, 3p)
                    const ulonglong2 tw = stw[v1 * 16 + o];
                    const u64 y = shoup_approx(r, tw.x, tw.y, np);        // [0, 4p)
                    const u32 a = w2 + (o >> 3) * 16384 + (o & 7) * 2048;
                    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(y) : "memory");
                }
            }
        }
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        // ---- round 2
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int t = 0; t < 2; t++)
#pragma unroll
                for (int s = 0; s < 4; s++)
                    tc_mma_i8(tmem + t * 128, tc_desc(sv_a + t * 16384 + s * 256, 128, 1024),
                              tc_desc(img2_a + s * 256, 128, 1024), idesc, s > 0 ? 1u : 0u);
            tc_commit(smem_u32(&mbar));
        }
        mbar_wait(smem_u32(&mbar), phase);
        phase ^= 1;
        tc_fence_after();
        {
            ulonglong2 sc = make_ulonglong2(0, 0);
            if (!FWD) sc = A.scale ? A.scale[b % A.scale_mod] : A.ninv[prime];
            const u32 m = 32 * q + lane, v2 = 8 * mtl + (m >> 4), c = m & 15;
            u64 *dst = A.out + (size_t)A.map.sout[b] * N + c0 + c;
#pragma unroll
            for (u32 o0 = ob; o0 < ob + NC_OUT; o0 += NC_ILP) {
                u32 v[NC_ILP][8];
#pragma unroll
                for (int k = 0; k < NC_ILP; k++) tc_ld8(tb + (o0 + k) * 8, v[k]);
                tc_wait_ld();
#pragma unroll
                for (int k = 0; k < NC_ILP; k++) {
                    const u32 o = o0 + k;
                    u64 r = bytesum_reduce_c<true>(v[k], np, mu);
                    if (!FWD) r = csub(csub(shoup_approx(r, sc.x, sc.y, np), 2 * pc.p), pc.p);
                    dst[(size_t)row2(v2, o) * 256] = r;
                }
            }
        }
        tc_fence_before();
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

hks_status launch_ntt_cols_tc(const hks_ctx *ctx, NttDir dir, int /*epi*/, const NttArgs &na, cudaStream_t s) {
    constexpr size_t smem = 98304 + 4096;
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
    const u32 grid = std::min<u32>(a.nlimbs * 16, 2 * (u32)nsm);
    ProfScope ps(dir == NTT_FWD ? K_NTT_FWD_COLS : K_NTT_INV_COLS, s);
    const cudaError_t e = dir == NTT_FWD
                              ? hks_launch(k_ntt_cols_tc<true>, dim3(grid), dim3(NC_THREADS), smem, s, a)
                              : hks_launch(k_ntt_cols_tc<false>, dim3(grid), dim3(NC_THREADS), smem, s, a);
    const double nn = 65536.0;
    ps.done(2.0 * a.nlimbs * nn * 8.0, a.nlimbs * (nn / 2.0) * 8 * 7.0);
    if (e != cudaSuccess) HKS_FAIL(HKS_ECUDA, "k_ntt_cols_tc launch: %s", cudaGetErrorString(e));
    return HKS_OK;
}
#else
hks_status launch_ntt_cols_tc(const hks_ctx *, NttDir, int, const NttArgs &, cudaStream_t) {
    HKS_FAIL(HKS_EINVAL, "tensor-core NTT column pass: experimental build only (HKS_EXPERIMENTAL=1)");
}
#endif  // HKS_EXPERIMENTAL
