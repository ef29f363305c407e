// internal.h -- context layout, kernel argument blocks and launcher declarations for libhks.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hks.h"
#include "modarith.cuh"

#ifndef HKS_EXPERIMENTAL
#define HKS_EXPERIMENTAL 0   // 1: also build the measured-and-rejected kernel variants and
#endif                       //    their environment switches (tools/build_variant.sh); never the product

#ifndef HKS_TW_PERSIST
#define HKS_TW_PERSIST 0       // 1: L2 access-policy window (persisting) over the twiddle tables
#endif
#ifndef HKS_KEY_STREAM
#define HKS_KEY_STREAM 0       // 1: key words loaded with the streaming (evict-first) cache hint
#endif
#ifndef HKS_NTT_TC_DEFAULT
#define HKS_NTT_TC_DEFAULT 0   // log N = 16 column passes on the tensor cores (ntt_tc.cu); 0: butterfly passes
#endif

typedef uint16_t u16;
typedef uint8_t u8;

// ----------------------------------------------------------------------------------------------
// Limb batches.  One kernel launch transforms up to HKS_MAXB limbs of N words; limb b reads slot
// sin[b] of the input base pointer and writes slot sout[b] of the output base pointer (slot s =
// words [s*N, (s+1)*N)), reduced modulo prime index prime[b].  The map travels in the kernel's
// parameter space (warp-uniform, constant-bank broadcast: §3.5).
#define HKS_MAXB 256

struct LimbMap {
    u16 sin[HKS_MAXB];
    u16 sout[HKS_MAXB];
    u16 prime[HKS_MAXB];
    u16 sa[HKS_MAXB];   // epilogue operand slot (ModDown: acc limb)
    u16 sb[HKS_MAXB];   // epilogue operand slot (ModDown: c0 limb), 0xffff = none
    uint8_t ob[HKS_MAXB];   // EPI_MODDOWN: output-table entry of limb b
};

#define NTT_MAXO 16         // output-table entries per ModDown launch

enum NttEpi : int {
    EPI_LAZY = 0,      // first pass: store lazily reduced values
    EPI_CANON = 1,     // last forward pass: canonical store
    EPI_MODDOWN = 2,   // last forward pass: out = (a - x) * P^-1 [+ b]  (PAPER.md:350 ModDown fusion)
    EPI_SCALE = 3,     // last inverse pass: out = x * s (s = N^-1 or N^-1 * qhat^-1) canonical
    EPI_TENSOR = 4,    // first inverse pass (rows) of d2 = in * in2, d2 also stored to side (HMult)
    EPI_MDTENSOR = 5,  // EPI_MODDOWN + tensor terms: role 0 adds a0*b0, role 1 adds a0*b1 + a1*b0
    EPI_SWITCH = 6,    // first forward pass (columns) of centered SwitchModulo(in) from sw_q (Rescale)
    EPI_LAZY_CIN = 7,  // first forward pass (columns), input in the coefficient-chunked layout (below)
    EPI_SCALE_COUT = 8 // last inverse pass (columns) as EPI_SCALE, output in the coefficient-chunked layout
};
// Coefficient-chunked layout (all-to-all limb sharding, shard.cu): coefficient x = r C + c of slot s lives at
// (r >> clog) * cstride + s * (C << clog) + (r & (2^clog - 1)) C + c, i.e. chunk k = rows [k 2^clog,
// (k + 1) 2^clog) of every limb, chunk-major.

struct NttArgs {
    const u64 *in;
    u64 *out;
    const PrimeConst *pc;      // per prime
    const ulonglong2 *tw;      // COLS: [nprimes][R] ; ROWS: [nprimes][R][C]   (w, w') pairs
    const ulonglong2 *tw2;     // single-pass cluster INTT (k_intt_cl): the column table; tw = the row table
    const ulonglong2 *scale;   // EPI_SCALE: per-limb (w, w') = scale[b % scale_mod]; NULL -> ninv[prime]
    const ulonglong2 *ninv;    // per prime N^-1
    const u64 *ea;             // EPI_MODDOWN operand a base (acc)
    const u64 *eb;             // EPI_MODDOWN operand b base (c0), may be NULL
    const ulonglong2 *pinv;    // per prime P^-1 mod q (Shoup)
    u64 galois;                // unused (kept for layout); see ogal
    // EPI_MODDOWN output table: limb b writes outs[ob[b]] and adds adds[ob[b]] read through ogal[ob[b]]
    u64 *outs[NTT_MAXO];
    const u64 *adds[NTT_MAXO];
    u64 ogal[NTT_MAXO];
    // EPI_TENSOR: second factor and the side output of the product (same slots as in / sin)
    const u64 *in2;
    u64 *side;
    // EPI_MDTENSOR: ciphertext halves (slot = output limb sout), role of output-table entry
    const u64 *ta0, *ta1, *tb0, *tb1;
    uint8_t trole[NTT_MAXO];
    // EPI_SWITCH: source modulus and sw_qmod[prime] = sw_q mod prime
    u64 sw_q;
    const u64 *sw_qmod;
    u32 log_n, log_r, log_c;   // N = R * C; R = 2^log_r rows, C = 2^log_c columns (row length)
    u32 clog;                  // EPI_LAZY_CIN / EPI_SCALE_COUT: log2 rows per chunk
    u64 cstride;               //   and words per chunk of the whole buffer
    u32 tiles;                 // CTAs per limb
    u32 scale_mod;
    u32 nlimbs;
    LimbMap map;
};

// ----------------------------------------------------------------------------------------------
// Base conversion (Eq. 1).  A group converts nsrc canonical y_i limbs to up to BC_MAXDST targets.
#define BC_MAXSRC 16
#define BC_MAXDST 64
#define BC_MAXG 16

struct BconvGroup {
    u32 nsrc, ndst, mat_stride;
    const uint2 *mat;          // [nsrc][mat_stride] (lo30, hi30) of [qhat_i]_t, column u = target u
    const double *matf;        // same entries as three exact 20-bit limbs [nsrc][mat_stride][3] (FP64 path) or NULL
    const u32 *mats;           // (lo30 + hi30) of each entry [nsrc][mat_stride] (Karatsuba path) or NULL
    const u64 *mimg;           // k_bconv_tc: shared-memory image of the B operand from this group's first target
                               // on (bconv_img_words(nsrc) words per target; see ctx.cu) or NULL
    const u64 *matb;           // byte-column words [nsrc][mat_stride][8] (tensor-pipe path, k_bconv_mma) or NULL:
                               // word c of entry (i, u) has byte a = byte c of (2^(8a) [qhat_i]_t mod t)
    u16 src_slot[BC_MAXSRC];
    const u64 *srcp[BC_MAXSRC];   // non-NULL: absolute address of source i (e.g. a peer GPU's limb over
                                  // NVLink, limb-sharded KeySwitch); NULL: in + src_slot[i] * N
    u16 src_prime[BC_MAXSRC];
    u16 dst_slot[BC_MAXDST];
    u16 dst_prime[BC_MAXDST];
};

// k_bconv_tc B operand: per target, NCH = 2 ceil(nsrc / 4) K-chunks of 8 rows (byte columns c) x 16
// bytes (words (2kc, t, c), (2kc + 1, t, c)), i.e. the canonical no-swizzle K-major UMMA layout
__host__ __device__ constexpr u32 bconv_img_words(u32 nsrc) { return 2 * ((nsrc + 3) / 4) * 16; }

#define NTT16_IMG 2048   // words per 16 x 16 column-pass matrix image (bconv_img_words(16) * 16 targets)
#define NTT16_TAB (2 * NTT16_IMG + 512)   // per prime: round-1 image, round-2 image, twist (w, w')[16][16]

// base + off, or NULL for an absent (not uploaded) table
template <typename T>
inline T *tab_at(T *base, size_t off) { return base ? base + off : nullptr; }

// host helpers (ctx.cu): the byte-column words of a matrix entry v = [qhat]_t (8 words, word c holding
// byte c of 2^(8a) v mod t in its byte a) and the k_bconv_tc image of a [nsrc][ntg][8] word table
void push_bytecols(std::vector<u64> &out, u64 v, u64 t);
void bconv_image(const u64 *matb, u32 nsrc, u32 ntg, std::vector<u64> &out);

struct BconvArgs {
    const u64 *in;
    u64 *out;
    const PrimeConst *pc;
    u32 log_n;
    u32 ngroups;
    u32 lazy_out;              // 1: outputs in [0, 8t) (consumer: forward NTT), 0: canonical
    u32 big;                   // 1: every prime > 2^49 (required by the tensor-pipe kernels k_bconv_tc / _mma)
    u32 cw;                    // k_bconv_mma: coefficients per CTA (set by the launcher)
    u32 fresh_tables;          // 1: mat / mimg were written by a kernel earlier on this stream (hks_bconv), so
                               // the tensor-core kernel, which stages them before griddepcontrol.wait, is
                               // launched without programmatic dependent launch
    BconvGroup g[BC_MAXG];
};

// ----------------------------------------------------------------------------------------------
// Key inner product (dot-product fusion).
struct KipArgs {
    const u64 *ext;    // [beta][ne][N]
    const u64 *c1;     // own-digit limbs read from here when non-NULL (KeySwitch), else from ext
    const u64 *evk;    // [dnum][2][nk][N]
    u64 *acc;          // [2][ne][N]
    const PrimeConst *pc;
    u64 galois;
    u32 log_n, level, nq, np, ne, nk, beta, alpha;
};

// Key inner product for several ciphertexts sharing one key (hoisted rotation batches): every key
// word is loaded once and applied to all nct ciphertexts.
#define KIP_MAXCT 8
struct KipMultiArgs {
    const u64 *ext[KIP_MAXCT];   // per ciphertext [beta][ne][N]
    const u64 *c1[KIP_MAXCT];    // per ciphertext own-digit source (EVAL)
    u64 *acc[KIP_MAXCT];         // per ciphertext [2][ne][N]
    const u64 *evk;
    const PrimeConst *pc;
    u64 galois;
    u32 nct, log_n, level, nq, np, ne, nk, beta, alpha;
};
hks_status launch_kip_multi(const KipMultiArgs &a, cudaStream_t s);

// ----------------------------------------------------------------------------------------------
// Fused last forward NTT pass + key inner product (PAPER.md:351 HMult fusion part (ii): "the NTT
// kernels generate NTT(x') * ksk"; PAPER.md:352 dot-product fusion).  Output limb u of a launch:
// for every digit j, D_j = row pass of ext slot dsrc[u][j] (pass-1 output), or -- bit 15 set --
// the already-EVAL limb c1[dsrc & 0x7fff] (own-digit limb); acc_p[aslot] = sum_j D_j * evk[j][p][kslot].
#define FK_MAXU 64
#define FK_MAXD 4
#define FK_DIRECT 0x8000

struct FusedKipMap {
    u16 prime[FK_MAXU];
    u16 kslot[FK_MAXU];
    u16 aslot[FK_MAXU];
    u16 dsrc[FK_MAXU][FK_MAXD];   // per term i: transformed terms first (i < ntr), then direct ones
    u8 dig[FK_MAXU][FK_MAXD];     // key digit j of term i
    u8 ntr[FK_MAXU];              // number of transformed terms of limb u (<= the launch's NTR)
    u16 yslot[FK_MAXU];           // 0xffff, or: write INTT row pass of acc_p to y slot p * ystride + yslot
};

struct FusedKipArgs {
    const u64 *ext;
    const u64 *c1;
    const u64 *evk;     // [dnum][2][nkey][N]
    u64 *acc;           // poly p, slot a at (p * acc_stride + a) * N
    const PrimeConst *pc;
    const ulonglong2 *tw;   // forward row twiddles [nprimes][R][C]
    u32 log_n, log_r, log_c, tiles, nu, ndig, nkey, acc_stride;
    u32 ntr;                // thread groups = max transformed terms over the launch
    u64 *y;                 // ModDown input buffer (y mode): first inverse-NTT pass of acc's P limbs
    const ulonglong2 *tw_inv;   // inverse row twiddles [nprimes][R][C]
    u32 ystride;
    FusedKipMap map;
};

hks_status launch_ntt_kip(const hks_ctx *ctx, FusedKipArgs &a, cudaStream_t s);

// ----------------------------------------------------------------------------------------------
// Fused plaintext-weighted sum of ciphertexts ("weighed sum ... 4n-2 down to n+1 memory
// operations"): out_p[t] = (accumulate ? out_p[t] : 0) + sum_j w_j[t] * x_{j,p}[t] (mod q_t), limbs
// t = 0..nlimbs-1 of the chain, one 128-bit 30-bit-split accumulation and one reduction per output.
#define WS_MAXT 16
struct WsumArgs {
    const u64 *w[WS_MAXT];
    const u64 *x0[WS_MAXT];
    const u64 *x1[WS_MAXT];
    u64 *out0, *out1;
    const PrimeConst *pc;
    u32 nterm, nlimbs, log_n, accumulate;
};
hks_status launch_pt_wsum(const WsumArgs &a, cudaStream_t s);
// out_p += r_p (mod q_t) for p = 0, 1 over nlimbs chain limbs (BSGS giant-step accumulation)
hks_status launch_add_ct(const u64 *r0, const u64 *r1, u64 *out0, u64 *out1, u32 nlimbs, u32 log_n,
                         const PrimeConst *pc, cudaStream_t s);

// One output limb of the fused row pass + key product: its prime, key slot, acc slot, and per digit j
// the source slot (ext pass-1 output, or FK_DIRECT | c1 slot for the own-digit limb).
struct KipItem {
    u16 prime, kslot, aslot;
    u16 src[FK_MAXD];
    u16 yslot = 0xffff;     // P limb whose acc goes straight into ModDown's inverse row pass
};
// Groups items by their number of transformed terms and launches k_ntt_kip per group.
hks_status run_ntt_kip(const hks_ctx *ctx, const std::vector<KipItem> &items, u32 ndig, const u64 *ext,
                       const u64 *c1, const u64 *evk, u64 *acc, u32 nkey, u32 acc_stride, cudaStream_t s,
                       u64 *y = nullptr, u32 ystride = 0);

// ----------------------------------------------------------------------------------------------
struct hks_ctx {
    u32 log_n, n, log_r, log_c, nq, np, dnum, alpha;
    int device;
    bool all_big = true;        // every prime > 2^49 (tensor-pipe base conversion)
    std::vector<u64> primes, psi;

    // host mirrors of the small tables (offsets into the device arrays)
    std::vector<size_t> mu_mat_off;     // [(L+1) * dnum]: matrix offset of (level, digit)
    std::vector<size_t> mu_scale_off;   // [L+1]: scale offset of level (ℓ+1 entries)

    // device tables (owned)
    PrimeConst *d_pc = nullptr;
    ulonglong2 *d_tw_col_fwd = nullptr, *d_tw_row_fwd = nullptr;   // all four inside d_tw_all (one allocation)
    ulonglong2 *d_tw_col_inv = nullptr, *d_tw_row_inv = nullptr;
    ulonglong2 *d_tw_all = nullptr;
    // L2 access-policy window over d_tw_all (num_bytes = 0: none): the NTT kernels' twiddle reads persist in
    // L2 while the key stream passes through (HKS_TW_PERSIST)
    cudaAccessPolicyWindow tw_win = {};
    ulonglong2 *d_ninv = nullptr;
    ulonglong2 *d_mu_scale = nullptr;   // ModUp: N^-1 * qhat_{j,i}^-1 mod q_i per (level, i)
    uint2 *d_mu_mat = nullptr;          // ModUp: [qhat_{j,i}]_t split, per (level, digit)
    ulonglong2 *d_md_scale = nullptr;   // ModDown: N^-1 * phat_k^-1 mod p_k  [K]
    uint2 *d_md_mat = nullptr;          // ModDown: [phat_k]_{q_i} split  [K][L+1]
    double *d_mu_matf = nullptr;        // ModUp matrices as 20-bit limbs in doubles (3 per entry)
    u32 *d_mu_mats = nullptr;           // ModUp matrices: lo30 + hi30 per entry (Karatsuba middle term)
    u32 *d_md_mats = nullptr;           // ModDown matrix: lo30 + hi30 per entry
    double *d_md_matf = nullptr;        // ModDown matrix as 20-bit limbs in doubles
    u64 *d_mu_matb = nullptr;           // ModUp matrices as byte-column words, 8 per entry (k_bconv_mma)
    u64 *d_md_matb = nullptr;           // ModDown matrix as byte-column words, 8 per entry
    std::vector<size_t> mu_img_off;     // [(L+1) * dnum]: word offset of the (level, digit) B image in d_mu_img
    u64 *d_mu_img = nullptr;            // ModUp matrices as k_bconv_tc B-operand images (per target contiguous)
    u64 *d_md_img = nullptr;            // ModDown matrix as a k_bconv_tc B-operand image
    // k_ntt_cols_tc (log N = 16): per prime NTT16_TAB words -- the B-operand images of the two 16-point
    // rounds of the column pass and the twist between them (ctx.cu, ntt_tc.cu)
    u64 *d_ntt_img_fwd = nullptr, *d_ntt_img_inv = nullptr;
    ulonglong2 *d_pinv = nullptr;       // P^-1 mod q_i  [L+1] (Shoup)
    // the ModDown matrix with P^-1 folded in, [phat_k P^-1]_{q_i}, for keys from hks_evk_prepare (whose Q limbs
    // carry the P^-1): the same layouts as d_md_mat / _mats / _matf / _matb / _img
    uint2 *d_mdp_mat = nullptr;
    u32 *d_mdp_mats = nullptr;
    double *d_mdp_matf = nullptr;
    u64 *d_mdp_matb = nullptr;
    u64 *d_mdp_img = nullptr;
    u64 *d_qmod = nullptr;              // Rescale: q_j mod q_i  [L+1][L+1] (row j = dropped limb)
    ulonglong2 *d_qlinv = nullptr;      // Rescale: q_j^-1 mod q_i (Shoup)  [L+1][L+1]

    // side streams for independent branches inside one call (the giant steps of hks_linear_transform):
    // created with the context, forked from / joined to the caller's stream with the events below; the
    // mutex serialises concurrent callers' enqueue phases (a wait binds the event's latest record)
#ifndef HKS_NSIDE
#define HKS_NSIDE 3   // side streams per context (measured: 1 / 2 / 3 -> C5 56.0 / 56.1 / 56.8 seq/s)
#endif
    static constexpr int NSIDE = HKS_NSIDE;
    cudaStream_t side[NSIDE] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[NSIDE] = {};
    mutable std::recursive_mutex side_mu;

    u32 L() const { return nq - 1; }
    u32 beta(u32 level) const { return (level + 1 + alpha - 1) / alpha; }
    u32 ne(u32 level) const { return level + 1 + np; }
    u32 digit_lo(u32 j) const { return j * alpha; }
    u32 digit_hi(u32 level, u32 j) const { u32 h = (j + 1) * alpha; return h < level + 1 ? h : level + 1; }
    u32 ext_prime(u32 level, u32 t) const { return t <= level ? t : nq + (t - level - 1); }
};

// ----------------------------------------------------------------------------------------------
// diagnostics (prof.cu): launch counter + optional per-launch event pair tagged with a kernel class
enum KCls { K_NTT_FWD_COLS = 0, K_NTT_FWD_ROWS, K_NTT_FWD_ROWS_MODDOWN, K_NTT_INV_ROWS, K_NTT_INV_COLS, K_BCONV,
            K_KIP, K_AUTOMORPH, K_NTT_ROWS_KIP, K_WSUM, K_ADD, K_NTT_INV_FUSED, K_NCLS };
struct ProfScope {
    int cls;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    ProfScope(int c, cudaStream_t st);
    // algorithmic_muls: 32x32->64-bit partial products the launch needs (4 per exact 60x60-bit
    // product; 7 wide-equivalents per Shoup butterfly: 3 for the quotient, 2 + 4/2 for the remainder)
    void done(double algorithmic_bytes, double algorithmic_muls = 0);
};

// ----------------------------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+): every kernel lets its stream successor launch as soon as all
// of its CTAs are running (pdl_trigger) and waits for its predecessor's completion and memory
// (pdl_wait) before touching anything the predecessor wrote, so a kernel's launch, CTA rasterisation
// and constant-table prologue overlap the previous kernel's tail.  HKS_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
// Per-(device, kernel) one-time setup, thread-safe: cudaFuncSetAttribute acts on the current device only,
// so a process with contexts on several devices raises each kernel's dynamic shared-memory limit once per
// device.  hks_num_sms: SM count of the current device (cached per device).
void hks_func_smem(const void *fn, size_t smem);
int hks_num_sms();
// per-kernel profiling on (hks_prof_enable): calls with independent branches then keep them on the caller's
// stream, so each launch's event pair times that kernel alone rather than its overlap with a sibling
bool prof_active();
// pdl = false: an ordinary stream-ordered launch, for a kernel whose pre-wait prologue reads tables a
// recent kernel of the same stream wrote (hks_bconv's device-built constants)
// win != NULL with num_bytes > 0: the launch carries that L2 access-policy window
template <typename... KArgs, typename... Args>
inline cudaError_t hks_launch_ex(bool pdl, const cudaAccessPolicyWindow *win, void (*kernel)(KArgs...), dim3 grid,
                                 dim3 block, size_t smem, cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.numAttrs = 1;
    if (win && win->num_bytes) {
        at[1].id = cudaLaunchAttributeAccessPolicyWindow;
        at[1].val.accessPolicyWindow = *win;
        cfg.numAttrs = 2;
    }
    cfg.attrs = at;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t hks_launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t s, Args &&...args) {
    return hks_launch_ex(pdl, nullptr, kernel, grid, block, smem, s, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t hks_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
    return hks_launch_pdl(pdl_enabled(), kernel, grid, block, smem, s, std::forward<Args>(args)...);
}

// ----------------------------------------------------------------------------------------------
// error plumbing
void hks_set_error(const char *fmt, ...);
#define HKS_FAIL(code, ...) do { hks_set_error(__VA_ARGS__); return code; } while (0)
#define HKS_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) HKS_FAIL(HKS_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    } while (0)
#define HKS_CHECK_LAUNCH() HKS_CUDA(cudaGetLastError())

// ----------------------------------------------------------------------------------------------
// launchers (ntt.cu, kernels.cu)
enum NttDir { NTT_FWD = 0, NTT_INV = 1 };
// pass 0 = first pass, pass 1 = second pass (forward: columns then rows; inverse: rows then columns)
hks_status launch_ntt_pass(const hks_ctx *ctx, NttDir dir, int pass, int epi, NttArgs &a, cudaStream_t s);
// full transform of a limb batch through both passes (in -> out, may alias), chunks > HKS_MAXB
struct LimbList {
    std::vector<u16> sin, sout, prime, sa, sb;
    void push(u32 i, u32 o, u32 p, u32 a = 0, u32 b = 0xffff) {
        sin.push_back((u16)i); sout.push_back((u16)o); prime.push_back((u16)p);
        sa.push_back((u16)a); sb.push_back((u16)b);
    }
    size_t size() const { return sin.size(); }
};
// in2 != NULL (inverse only): the first pass transforms in * in2 (tensor term) and stores the product
// to side (same slots as in).
hks_status run_ntt(const hks_ctx *ctx, NttDir dir, const LimbList &L, const u64 *in, u64 *out,
                   const ulonglong2 *scale, u32 scale_mod, cudaStream_t s, const u64 *in2 = nullptr,
                   u64 *side = nullptr);
// second (column) pass of the inverse NTT only (the row pass was fused into k_ntt_kip)
hks_status run_ntt_inv_cols(const hks_ctx *ctx, const LimbList &L, const u64 *in, u64 *out, const ulonglong2 *scale,
                            u32 scale_mod, cudaStream_t s);
// first (column) pass of the forward NTT only; the row pass is fused elsewhere (launch_ntt_kip)
hks_status run_ntt_fwd_cols(const hks_ctx *ctx, const LimbList &L, const u64 *in, u64 *out, cudaStream_t s);
// ModDown's last NTT + epilogue for many polynomials at once: limb i of L belongs to polynomial
// poly[i]; polynomial p writes outs[p] (+ adds[p] through the automorphism gal[p]).
struct MdOut {
    u64 *out;
    const u64 *add;
    u64 galois;
};
// tensor != NULL (HMult): {a0, a1, b0, b1}; polynomial 0 adds a0 b0, polynomial 1 adds a0 b1 + a1 b0.
// cin != NULL: the column pass reads limb i from the coefficient-chunked buffer cin (slot cin_slot[i], clog,
// cstride) instead of buf, and writes buf slot L.sin[i].
struct ChunkIn {
    const u64 *buf;
    u32 clog;
    u64 cstride;
    std::vector<u16> slot;
};
hks_status run_ntt_moddown(const hks_ctx *ctx, const LimbList &L, const std::vector<uint8_t> &poly,
                           const std::vector<MdOut> &outs, u64 *buf, const u64 *acc, cudaStream_t s,
                           const u64 *const *tensor = nullptr, const ChunkIn *cin = nullptr, bool prepared = false);
// Rescale of npoly polynomials (top limbs already COEFF in coef slots 0..npoly-1), see ntt.cu.
hks_status run_rescale(const hks_ctx *ctx, u32 npoly, u32 level, const u64 *x, const u64 *coef, u64 *buf,
                       u64 *const *outs, cudaStream_t s);
hks_status launch_bconv(const BconvArgs &a, u32 max_ndst, cudaStream_t s);
// column pass of the log N = 16 NTT on the tensor cores (ntt_tc.cu k_ntt_cols_tc): forward EPI_LAZY or
// inverse EPI_SCALE, same limb map / scale semantics as launch_ntt_pass
hks_status launch_ntt_cols_tc(const hks_ctx *ctx, NttDir dir, int epi, const NttArgs &a, cudaStream_t s);
bool ntt_tc_enabled();
bool bconv_tc_enabled();
bool bconv_tc_large(u32 log_n, u32 ngroups);
// out[i] = in[i] * w_i mod p_i (canonical) for n <= 16 limbs (hks_bconv's y_i = x_i [qhat_i]^-1)
// dw (device): w[0..nl) then the Shoup companions wp[0..nl); p (host): the limbs' primes
hks_status launch_limb_scale(const u64 *in, u64 *out, u32 nl, const u64 *dw, const u64 *p, u32 log_n, cudaStream_t s);
hks_status launch_evk_prepare(const hks_ctx *c, const u64 *in, u64 *out, u32 ndig, cudaStream_t s);
// hks_bconv's Eq. 1 constants for one (src, dst) pair, derived on the device (kernels.cu k_bconv_prep):
// w = [qhat_i^-1]_{q_i} and Shoup companions (2 nsrc words), mat [nsrc][ndst] (lo30, hi30) of [qhat_i]_t,
// the k_bconv_tc B image img [ndst][bconv_img_words(nsrc)]
hks_status launch_bconv_prep(const u64 *src, u32 nsrc, const u64 *dst, u32 ndst, u64 *w, uint2 *mat, u64 *img,
                             cudaStream_t s);
hks_status launch_kip(const KipArgs &a, cudaStream_t s);
hks_status launch_automorph(const u64 *in, u64 *out, u32 nlimbs, u32 log_n, u64 galois, cudaStream_t s);
