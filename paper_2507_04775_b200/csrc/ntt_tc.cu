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
// D in TMEM, one byte-sum reduction per output (modarith.cuh bytesum_reduce_c: mostly ALU-pipe work).  Per
// element that is two reductions and one Shoup product (the twist) instead of the four butterfly Shoup
// products of the butterfly pass, so the pass can run at the HBM rate of its 16 bytes per element.
//
// A tile = (limb, 8 columns): 128 vectors per round = one M = 128 MMA of K = 128 (four k32 steps).  The
// kernel is persistent (one CTA per SM, contiguous balanced tile ranges, so a CTA meets one or two limbs)
// and warp-specialised, every hand-off an mbarrier:
//   warp 0      TMA producer: one 4-D tensor copy per tile (8 columns x 16 x 16 rows = 16 KB) into NC_S
//               shared stages, and the two matrix images of each new prime (1-D bulk copy, 32 KB) into one
//               of two table slots;
//   warp 1      TMEM owner and MMA issuer (one thread): round 1 of tile j with its A operand in TMEM
//               (kind::i8, A from tensor memory), then round 2 of tile j - 1 from shared memory;
//   warps 2-5   transposers (one per TMEM lane quarter): a thread = one round-1 vector, 16 conflict-free
//               8-byte shared loads -> 32 registers -> one tcgen05.st into the round-1 A operand;
//   warps 6-13  round-1 epilogue: TMEM -> reduce -> twist (Shoup pairs held in registers) -> round 2's A
//               operand in shared memory (256 contiguous bytes per warp store);
//   warps 14-17 round-2 epilogue: TMEM -> reduce (-> scale) -> global stores.
// Outputs are congruent to the butterfly pass's: forward lazily reduced to [0, 3p) (the row pass accepts
// [0, 8p + 2^32)), inverse scaled and canonical.  Parity: every KeySwitch / HMult / NTT test runs through
// this pass when it is the default (HKS_NTT_TC_DEFAULT).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "internal.h"
#include "tc.cuh"

#define NC_CW 8                 // columns per tile
#define NC_TPL (256 / NC_CW)    // tiles per limb
#ifndef NC_CPT
#define NC_CPT 4                // tiles per TMA stage (a chunk of NC_CPT * 8 adjacent columns)
#endif
#define NC_SW (NC_CW * NC_CPT)  // columns per stage: NC_SW * 8-byte row segments per TMA box row
#ifndef NC_S
#define NC_S 2                  // TMA stages
#endif
#define NC_STAGE (16384 * NC_CPT)   // bytes of one stage (256 rows x NC_SW words)
#define NC_OPB 16384            // bytes of one round-2 operand buffer (128 vectors x 128 bytes)
#define NC_TABB 32768           // bytes of one table slot (round-1 and round-2 images)
#define NC_NW 19                // warps: producer, MMA round 1, 4 transposers, 8 + 4 epilogue, MMA round 2
                                // (<= 5 warps per SM sub-partition keeps 96 registers per thread)
#define NC_THREADS (NC_NW * 32)
#define NC_W_TR 2
#define NC_W_E1 6
#define NC_W_E2 14
#define NC_W_M2 18
#define NC_SMEM (NC_S * NC_STAGE + 2 * NC_OPB + 2 * NC_TABB + 1024)
// TMEM columns: D1 x2 [0, 256), D2 [256, 384), A1 x2 [384, 448)
#define NC_D2 256
#define NC_A1 384

struct NttColsArgs {
    CUtensorMap tmap;           // 4-D view of the input (columns, two 16-row digits, slot); box 8 x 16 x 16 x 1
    u64 *out;
    const u64 *tab;             // [prime][NTT16_TAB]: round-1 image, round-2 image, twist (w, w')[16][16]
    const ulonglong2 *scale;    // inverse: scale[b % scale_mod] or, if NULL, ninv[prime]
    const ulonglong2 *ninv;
    const PrimeConst *pc;
    u32 nlimbs, scale_mod;
    LimbMap map;
#ifdef NC_TRACE
    long long *trace;           // [event][tile] clock64 stamps of CTA 0 (debug builds)
#endif
};
#ifdef NC_TRACE
#define NC_T(ev, j) do { if (blockIdx.x == 0 && (j) < 64) A.trace[(ev) * 64 + (j)] = clock64(); } while (0)
#else
#define NC_T(ev, j) do { } while (0)
#endif

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_mma_i8_ts(u32 dtmem, u32 atmem, u64 bdesc, u32 idesc, u32 accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
        "r"(atmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_st32(u32 taddr, const u32 (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    u32 pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <bool FWD>
__global__ void __launch_bounds__(NC_THREADS, 1) k_ntt_cols_tc(const __grid_constant__ NttColsArgs A) {
    pdl_trigger();
    constexpr u32 N = 1u << 16;
    extern __shared__ uint8_t csm_raw[];
    __shared__ __align__(8) u64 tma_full[NC_S], tma_empty[NC_S], img_full[2], img_free[2];
    __shared__ __align__(8) u64 a1_full[2], a1_empty[2], d1_full[2], d1_empty[2], a2_full[2], a2_empty[2];
    __shared__ __align__(8) u64 d2_full, d2_empty;
    __shared__ u32 tmem_s;
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const u32 nchunk = A.nlimbs * (NC_TPL / NC_CPT);
    const u32 ch_beg = (u32)((u64)blockIdx.x * nchunk / gridDim.x);    // balanced contiguous chunk ranges
    const u32 ch_end = (u32)((u64)(blockIdx.x + 1) * nchunk / gridDim.x);
    const u32 t_beg = ch_beg * NC_CPT;
    const u32 nloc = (ch_end - ch_beg) * NC_CPT;
    const u32 b_first = t_beg / NC_TPL;
    // table segment of local tile j: the limb offset from the CTA's first limb (slot = segment & 1)
    auto seg = [&](u32 j) { return (t_beg + j) / NC_TPL - b_first; };
    auto last_of_seg = [&](u32 j) { return j + 1 == nloc || seg(j + 1) != seg(j); };

    // 1024-aligned dynamic shared memory: stages | round-2 operands | table slots
    const u32 sbase = (smem_u32(csm_raw) + 1023) & ~1023u;
    const u32 stg0 = sbase, op2 = stg0 + NC_S * NC_STAGE, tab0 = op2 + 2 * NC_OPB;
    uint8_t *const sgen = csm_raw + (sbase - smem_u32(csm_raw));

    if (tid == 0) {
        for (int s = 0; s < NC_S; s++) {
            mbar_init(smem_u32(&tma_full[s]), 1);
            mbar_init(smem_u32(&tma_empty[s]), 4 * NC_CPT);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(smem_u32(&img_full[b]), 1);
            mbar_init(smem_u32(&img_free[b]), 1);
            mbar_init(smem_u32(&a1_full[b]), 4);
            mbar_init(smem_u32(&a1_empty[b]), 1);
            mbar_init(smem_u32(&d1_full[b]), 1);
            mbar_init(smem_u32(&d1_empty[b]), 8);
            mbar_init(smem_u32(&a2_full[b]), 8);
            mbar_init(smem_u32(&a2_empty[b]), 1);
        }
        mbar_init(smem_u32(&d2_full), 1);
        mbar_init(smem_u32(&d2_empty), 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const u32 tmem = tmem_s;
    if (warp != 0) pdl_wait();   // the producer waits after issuing its first table copy (ctx tables only)

    if (warp == 0) {
        // ---------------- TMA producer (warp-uniform loop, one elected lane issues) ----------------
        if (elect_one()) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<u64>(&A.tmap)) : "memory");
        for (u32 n = 0; n * NC_CPT < nloc; n++) {
            const u32 j = n * NC_CPT, s = n % NC_S;
            const u32 tile = t_beg + j, b = tile / NC_TPL, c0 = (tile % NC_TPL) * NC_CW;
            if (j == 0 || seg(j) != seg(j - 1)) {
                // the round-1 / round-2 images of a new limb's prime into slot seg & 1, after the last round-2
                // MMA of segment seg - 2 released it (ctx tables: no wait on the predecessor)
                const u32 k = seg(j);
                if (k >= 2) mbar_wait(smem_u32(&img_free[k & 1]), ((k - 2) >> 1) & 1);
                if (elect_one()) {
                    const u32 bar = smem_u32(&img_full[k & 1]);
                    mbar_expect_tx(bar, NC_TABB);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            tab0 + (k & 1) * NC_TABB),
                        "l"(A.tab + (size_t)A.map.prime[b] * NTT16_TAB), "r"((u32)NC_TABB), "r"(bar)
                        : "memory");
                }
                __syncwarp();
            }
            if (j == 0) pdl_wait();   // the tile data is the predecessor's output
            if (n >= NC_S) mbar_wait(smem_u32(&tma_empty[s]), ((n / NC_S) - 1) & 1);
            NC_T(0, j);
            if (elect_one()) {
                const u32 bar = smem_u32(&tma_full[s]);
                mbar_expect_tx(bar, NC_STAGE);
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3, %4, %5}], [%6];" ::"r"(stg0 + s * NC_STAGE),
                    "l"(reinterpret_cast<u64>(&A.tmap)), "r"(c0), "r"(0), "r"(0), "r"((u32)A.map.sin[b]), "r"(bar)
                    : "memory");
            }
            __syncwarp();
        }
    } else if (warp == 1 || warp == NC_W_M2) {
        // ---------------- MMA issuers: warp 1 round 1, warp NC_W_M2 round 2 ----------------
        // The whole warp runs the loop (its values stay warp-uniform, so the descriptors live in uniform
        // registers); one elected lane issues.  Descriptors: the 14-bit start-address field advances by 16
        // per 256-byte k32 step.
        constexpr u32 idesc = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);   // M = N = 128, s32 += u8 x u8
        const u64 db1_0 = tc_desc(tab0, 128, 1024), db1_1 = tc_desc(tab0 + NC_TABB, 128, 1024);
        const u64 db2_0 = tc_desc(tab0 + NC_TABB / 2, 128, 1024), db2_1 = tc_desc(tab0 + NC_TABB + NC_TABB / 2, 128, 1024);
        const u64 da2_0 = tc_desc(op2, 128, 1024), da2_1 = tc_desc(op2 + NC_OPB, 128, 1024);
        auto round2 = [&](u32 i) {
            const u32 s = i & 1;
            NC_T(11, i);
            mbar_wait(smem_u32(&a2_full[s]), (i >> 1) & 1);
            if (i >= 1) mbar_wait(smem_u32(&d2_empty), (i - 1) & 1);
            tc_fence_after();
            NC_T(12, i);
            const u64 a = s ? da2_1 : da2_0, bb = (seg(i) & 1) ? db2_1 : db2_0;
            if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; k++) tc_mma_i8(tmem + NC_D2, a + 16 * k, bb + 16 * k, idesc, k > 0 ? 1u : 0u);
                tc_commit(smem_u32(&a2_empty[s]));
                tc_commit(smem_u32(&d2_full));
                if (last_of_seg(i)) tc_commit(smem_u32(&img_free[seg(i) & 1]));
            }
            __syncwarp();
            NC_T(6, i);
        };
        if (warp == 1) {
            for (u32 j = 0; j < nloc; j++) {
                const u32 s = j & 1;
                NC_T(9, j);
                if (j == 0 || seg(j) != seg(j - 1)) mbar_wait(smem_u32(&img_full[seg(j) & 1]), (seg(j) >> 1) & 1);
                mbar_wait(smem_u32(&a1_full[s]), (j >> 1) & 1);
                if (j >= 2) mbar_wait(smem_u32(&d1_empty[s]), ((j >> 1) - 1) & 1);
                tc_fence_after();
                NC_T(10, j);
                const u64 bb = (seg(j) & 1) ? db1_1 : db1_0;
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        tc_mma_i8_ts(tmem + s * 128, tmem + NC_A1 + s * 32 + k * 8, bb + 16 * k, idesc, k > 0 ? 1u : 0u);
                    tc_commit(smem_u32(&a1_empty[s]));
                    tc_commit(smem_u32(&d1_full[s]));
                }
                __syncwarp();
                NC_T(3, j);
            }
        } else {
            for (u32 i = 0; i < nloc; i++) round2(i);
        }
    } else if (warp < NC_W_E1) {
        // ---------------- transposers: stage [r_hi][r_lo][c] -> round-1 A operand in TMEM ----------------
        // vector m = 8 v + c; its element k is stage word (16 k + v) NC_SW + 8 sub + c (the tensor map orders
        // the row digits so that k is the outer one in both directions; sub = the tile's place in its chunk)
        const u32 q = warp & 3, m = q * 32 + lane, v = m >> 3, c = m & 7;
        const u64 *stg = reinterpret_cast<const u64 *>(sgen);
        for (u32 j = 0; j < nloc; j++) {
            const u32 n = j / NC_CPT, s = n % NC_S, sub = j % NC_CPT;
            mbar_wait(smem_u32(&tma_full[s]), (n / NC_S) & 1);
            if (warp == NC_W_TR && lane == 0) NC_T(1, j);
            u32 r[32];
            const u64 *p = stg + (size_t)s * (NC_STAGE / 8) + v * NC_SW + sub * 8 + c;
#pragma unroll
            for (int k = 0; k < 16; k++) {
                const u64 x = p[k * 16 * NC_SW];
                r[2 * k] = (u32)x;
                r[2 * k + 1] = (u32)(x >> 32);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tma_empty[s]));
            const u32 sa = j & 1;
            if (j >= 2) mbar_wait(smem_u32(&a1_empty[sa]), ((j >> 1) - 1) & 1);
            tc_fence_after();
            tc_st32(tmem + NC_A1 + sa * 32 + ((q * 32) << 16), r);
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&a1_full[sa]));
            if (warp == NC_W_TR && lane == 0) NC_T(2, j);
        }
    } else if (warp < NC_W_E2) {
        // ---------------- round-1 epilogue: reduce, twist, round 2's operand ----------------
        const u32 ew = warp - NC_W_E1;
        const u32 q = warp & 3, half = ew >> 2;             // TMEM lane quarter; outputs [8 half, 8 half + 8)
        const u32 m = q * 32 + lane, v = m >> 3, c = m & 7;  // this lane's vector (class / block v, column c)
        for (u32 j = 0; j < nloc; j++) {
            const u32 b = (t_beg + j) / NC_TPL, prime = A.map.prime[b];
            const PrimeConst pc = A.pc[prime];
            const u64 np = 0 - pc.p;
            const u32 mu = (u32)pc.mu80;
            // twist pairs (w, w') of this lane's class and outputs (read-only path, L1-resident per prime)
            const ulonglong2 *tw = reinterpret_cast<const ulonglong2 *>(A.tab + (size_t)prime * NTT16_TAB + 2 * NTT16_IMG) +
                                   v * 16 + 8 * half;
            const u32 s = j & 1;
            mbar_wait(smem_u32(&d1_full[s]), (j >> 1) & 1);
            if (warp == NC_W_E1 && lane == 0) NC_T(4, j);
            tc_fence_after();
            if (j >= 2) mbar_wait(smem_u32(&a2_empty[s]), ((j >> 1) - 1) & 1);
            const u32 tb = tmem + s * 128 + ((q * 32) << 16) + 64 * half;
            // round-2 vector o * 8 + c, element v
            const u32 w2 = op2 + s * NC_OPB + (v >> 1) * 128 + c * 16 + (v & 1) * 8;
            // all eight outputs of this warp's half in flight at once (two 32-column TMEM loads)
            u32 r[2][32];
            tc_ld32(tb, r[0]);
            tc_ld32(tb + 32, r[1]);
            tc_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&d1_empty[s]));
            u64 x[8];
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const u32 *rr = &r[o >> 2][8 * (o & 3)];
                x[o] = bytesum_reduce_c<true>(rr[0], rr[1], rr[2], rr[3], rr[4], rr[5], rr[6], rr[7], np, mu);   // [0, 3p)
            }
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const ulonglong2 t = __ldg(tw + o);
                const u64 y = shoup_approx(x[o], t.x, t.y, np);                        // [0, 4p)
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(w2 + (8 * half + o) * 1024), "l"(y) : "memory");
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&a2_full[s]));
            if (warp == NC_W_E1 && lane == 0) NC_T(5, j);
        }
    } else {
        // ---------------- round-2 epilogue: reduce (scale), store ----------------
        const u32 q = warp & 3;
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
            mbar_wait(smem_u32(&d2_full), j & 1);
            if (warp == NC_W_E2 && lane == 0) NC_T(7, j);
            tc_fence_after();
            const u32 tb = tmem + NC_D2 + ((q * 32) << 16);
#pragma unroll
            for (u32 o0 = 0; o0 < 16; o0 += 8) {
                u32 r[2][32];
                tc_ld32(tb + o0 * 8, r[0]);
                tc_ld32(tb + o0 * 8 + 32, r[1]);
                tc_wait_ld();
                if (o0 == 8) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&d2_empty));
                }
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const u32 o = o0 + k;
                    const u32 *rr = &r[k >> 2][8 * (k & 3)];
                    u64 x = bytesum_reduce_c<true>(rr[0], rr[1], rr[2], rr[3], rr[4], rr[5], rr[6], rr[7], np, mu);
                    if (!FWD) x = csub(csub(shoup_approx(x, sc.x, sc.y, np), 2 * pc.p), pc.p);
                    const u32 row = FWD ? 16 * g + o : g + 16 * o;
                    dst[(size_t)row * 256] = x;
                }
            }
            if (warp == NC_W_E2 && lane == 0) NC_T(8, j);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

#ifdef NC_TRACE
long long *hks_nc_trace = nullptr;
extern "C" void *hks_debug_nc_trace() { return hks_nc_trace; }
#endif
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

hks_status launch_ntt_cols_tc(const hks_ctx *ctx, NttDir dir, int /*epi*/, const NttArgs &na, cudaStream_t s) {
    constexpr size_t smem = NC_SMEM;
    const int nsm = hks_num_sms();
    hks_func_smem((const void *)k_ntt_cols_tc<true>, smem);
    hks_func_smem((const void *)k_ntt_cols_tc<false>, smem);
    NttColsArgs a;
    a.out = na.out;
    a.tab = dir == NTT_FWD ? ctx->d_ntt_img_fwd : ctx->d_ntt_img_inv;
    a.scale = na.scale;
    a.ninv = ctx->d_ninv;
    a.pc = ctx->d_pc;
    a.nlimbs = na.nlimbs;
    a.scale_mod = na.scale_mod ? na.scale_mod : 1;
    a.map = na.map;
#ifdef NC_TRACE
    {
        static long long *tr = nullptr;
        if (!tr) cudaMalloc(&tr, 13 * 64 * sizeof(long long));
        a.trace = tr;
        hks_nc_trace = tr;
    }
#endif
    // input view: (column, row digit 1, row digit 2, slot); the digit whose index is the element index k of a
    // round-1 vector comes second so that the stage lands as [k][v][c] (forward: row = v + 16 k; inverse:
    // row = 16 v + k)
    u32 nslot = 0;
    for (u32 i = 0; i < na.nlimbs; i++) nslot = std::max<u32>(nslot, (u32)na.map.sin[i] + 1);
    PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
    if (!enc) HKS_FAIL(HKS_ECUDA, "ntt_cols_tc: cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[4] = {256, 16, 16, nslot};
    const cuuint64_t str[3] = {dir == NTT_FWD ? 2048ull : 32768ull, dir == NTT_FWD ? 32768ull : 2048ull, 524288ull};
    const cuuint32_t box[4] = {NC_SW, 16, 16, 1}, es[4] = {1, 1, 1, 1};
    const CUresult cr = enc(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<u64 *>(na.in), dims, str, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) HKS_FAIL(HKS_ECUDA, "ntt_cols_tc: cuTensorMapEncodeTiled failed (%d)", (int)cr);
    const u32 grid = std::min<u32>(a.nlimbs * (NC_TPL / NC_CPT), (u32)nsm);
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
