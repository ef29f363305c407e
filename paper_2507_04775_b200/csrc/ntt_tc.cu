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

#define NC_THREADS 256

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

// Shared memory (dynamic, 1024-aligned): [0, 64K) vector operands -- round 1: M-tile mt (classes
// 4mt..4mt+3 x 32 columns) at mt * 16K, K-major, SBO 1024; round 2: two K halves (elements 0-7 / 8-15)
// at 0 / 32K, M-tile mt2 at mt2 * 8K, SBO 512 -- [64K, 80K) round-1 image, [80K, 96K) round-2 image,
// [96K, 100K) twist.
template <bool FWD>
__global__ void __launch_bounds__(NC_THREADS, 2) k_ntt_cols_tc(const __grid_constant__ NttColsArgs A) {
    pdl_trigger();
    constexpr u32 N = 1u << 16;
    extern __shared__ __align__(1024) uint8_t csm[];
    uint8_t *sv = csm;
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
    const u32 sv_a = smem_u32(sv), img1_a = smem_u32(simg1), img2_a = smem_u32(simg2);
    u32 phase = 0;
    u32 cur_prime = 0xffffffffu;
    // round-1 / round-2 row of element k of vector class v:  strided v + 16k, blocked 16v + k
    auto row1 = [](u32 v, u32 k) { return FWD ? v + 16 * k : 16 * v + k; };
    auto row2 = [](u32 v, u32 k) { return FWD ? 16 * v + k : v + 16 * k; };

    const u32 ntile = A.nlimbs * 8;
    for (u32 tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const u32 b = tile >> 3, c0 = (tile & 7) * 32;
        const u32 prime = A.map.prime[b];
        const u64 *src = A.in + (size_t)A.map.sin[b] * N + c0;
        u64 *dst = A.out + (size_t)A.map.sout[b] * N + c0;
        // ---- load: the tile's 8192 words into the round-1 operand layout (+ the prime's tables)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const u32 V = tid + 256 * h;                  // vector: class V / 32, column V % 32
            const u32 mt = V >> 7, m = V & 127, cls = V >> 5, c = V & 31;
            const u32 base = sv_a + mt * 16384 + (m >> 3) * 1024 + (m & 7) * 16;
#pragma unroll
            for (int k = 0; k < 16; k++) cp_async8(base + (k >> 1) * 128 + (k & 1) * 8, src + (size_t)row1(cls, k) * 256 + c);
        }
        if (prime != cur_prime) {
            const uint8_t *t = reinterpret_cast<const uint8_t *>(A.tab + (size_t)prime * NTT16_TAB);
            for (u32 o = tid * 16; o < 36864; o += NC_THREADS * 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(img1_a + o), "l"(t + o) : "memory");
            cur_prime = prime;
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();

        const PrimeConst pc = A.pc[prime];
        const u64 np = 0 - pc.p;
        const u32 mu = (u32)pc.mu80;
        const u32 q = warp & 3, mtl = warp >> 2;          // TMEM lane quarter, M-tile of the pair
        // ---- round 1: two M-tile pairs; outputs twisted into round 2's operand layout
        for (u32 pr = 0; pr < 2; pr++) {
            if (tid == 0) {
                tc_fence_after();
#pragma unroll
                for (int t = 0; t < 2; t++)
#pragma unroll
                    for (int s = 0; s < 4; s++)
                        tc_mma_i8(tmem + t * 128, tc_desc(sv_a + (2 * pr + t) * 16384 + s * 256, 128, 1024),
                                  tc_desc(img1_a + s * 256, 128, 1024), idesc, s > 0 ? 1u : 0u);
                tc_commit(smem_u32(&mbar));
            }
            mbar_wait(smem_u32(&mbar), phase);
            phase ^= 1;
            tc_fence_after();
            const u32 v1 = 4 * (2 * pr + mtl) + q, c = lane;   // this thread's round-1 vector
            const u32 tb = tmem + mtl * 128 + ((q * 32) << 16);
            // round-2 operand: vector v2 = o (M-tile o / 4, row (o % 4) 32 + c), element v1
            const u32 half = v1 >> 3, kk = v1 & 7;
            const u32 w2 = sv_a + half * 32768 + (c >> 3) * 512 + (kk >> 1) * 128 + (c & 7) * 16 + (kk & 1) * 8;
#pragma unroll
            for (u32 o0 = 0; o0 < 16; o0 += 4) {
                u32 v[4][8];
#pragma unroll
                for (int k = 0; k < 4; k++) tc_ld8(tb + (o0 + k) * 8, v[k]);
                tc_wait_ld();
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const u32 o = o0 + k;
                    const u64 r = bytesum_reduce_c<true>(v[k], np, mu);   // [0, 3p)
                    const ulonglong2 tw = stw[v1 * 16 + o];
                    const u64 y = shoup_approx(r, tw.x, tw.y, np);        // [0, 4p)
                    const u32 a = w2 + (o >> 2) * 8192 + (o & 3) * 2048;
                    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(y) : "memory");
                }
            }
            tc_fence_before();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
        }
        // ---- round 2: two M-tile pairs; outputs to global
        ulonglong2 sc = make_ulonglong2(0, 0);
        if (!FWD) sc = A.scale ? A.scale[b % A.scale_mod] : A.ninv[prime];
        for (u32 pr = 0; pr < 2; pr++) {
            if (tid == 0) {
                tc_fence_after();
#pragma unroll
                for (int t = 0; t < 2; t++)
#pragma unroll
                    for (int s = 0; s < 4; s++)
                        tc_mma_i8(tmem + t * 128,
                                  tc_desc(sv_a + (s >> 1) * 32768 + (2 * pr + t) * 8192 + (s & 1) * 256, 128, 512),
                                  tc_desc(img2_a + s * 256, 128, 1024), idesc, s > 0 ? 1u : 0u);
                tc_commit(smem_u32(&mbar));
            }
            mbar_wait(smem_u32(&mbar), phase);
            phase ^= 1;
            tc_fence_after();
            const u32 v2 = 4 * (2 * pr + mtl) + q, c = lane;
            const u32 tb = tmem + mtl * 128 + ((q * 32) << 16);
#pragma unroll
            for (u32 o0 = 0; o0 < 16; o0 += 4) {
                u32 v[4][8];
#pragma unroll
                for (int k = 0; k < 4; k++) tc_ld8(tb + (o0 + k) * 8, v[k]);
                tc_wait_ld();
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const u32 o = o0 + k;
                    u64 r = bytesum_reduce_c<true>(v[k], np, mu);
                    if (!FWD) r = csub(csub(shoup_approx(r, sc.x, sc.y, np), 2 * pc.p), pc.p);
                    dst[(size_t)row2(v2, o) * 256 + c] = r;
                }
            }
            tc_fence_before();
            __syncthreads();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

hks_status launch_ntt_cols_tc(const hks_ctx *ctx, NttDir dir, int /*epi*/, const NttArgs &na, cudaStream_t s) {
    constexpr size_t smem = 98304 + 4096;
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_ntt_cols_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_ntt_cols_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
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
    const u32 grid = std::min<u32>(a.nlimbs * 8, 2 * (u32)nsm);
    ProfScope ps(dir == NTT_FWD ? K_NTT_FWD_COLS : K_NTT_INV_COLS, s);
    const cudaError_t e = dir == NTT_FWD
                              ? hks_launch(k_ntt_cols_tc<true>, dim3(grid), dim3(NC_THREADS), smem, s, a)
                              : hks_launch(k_ntt_cols_tc<false>, dim3(grid), dim3(NC_THREADS), smem, s, a);
    const double nn = 65536.0;
    ps.done(2.0 * a.nlimbs * nn * 8.0, a.nlimbs * (nn / 2.0) * 8 * 7.0);
    if (e != cudaSuccess) HKS_FAIL(HKS_ECUDA, "k_ntt_cols_tc launch: %s", cudaGetErrorString(e));
    return HKS_OK;
}
