/*
 * hks.h -- C ABI of libhks: CKKS hybrid key switching on NVIDIA B200 (sm_100a).
 *
 * The boundary follows the paper's statement of the problem (FIDESlib, arXiv 2507.04775,
 * /root/reference/PAPER.md): a Context built once from (N, the Q chain, the special primes P,
 * dnum) with all precomputation (§3.5), polynomials resident in GPU memory
 * (§3.2), and the server-side key-switching steps of §3.6.3-§3.6.6.
 * The operation list is SURVEY.md §8(b).
 *
 * Conventions (all entry points)
 *   Buffers   Every polynomial buffer is caller-owned CUDA device memory on the context's device,
 *             u64 little-endian, limb-major [limbs][N], residues canonical in [0, m) for the limb's
 *             prime m.  The library never allocates on a hot-path call; the caller sizes the
 *             workspace with hks_workspace_bytes().  evk buffers are borrowed for the call.
 *   Forms     EVAL = bit-reversed evaluation order: x[j] = a(psi^(2*brv(j)+1)) (PAPER.md:341:
 *             NTT output is bit-reversed, iNTT takes bit-reversed and returns natural order).
 *             COEFF = natural coefficient order.  psi = the minimal primitive 2N-th root of unity
 *             modulo each prime (SURVEY.md §8(c) reading 1; query it with hks_ctx_psi()).
 *   Primes    Prime index space: 0..num_q-1 = q_0..q_L, num_q..num_q+num_p-1 = p_0..p_{K-1}.
 *             Extended limb order at level l: Q_0..Q_l, P_0..P_{K-1}.  Key limb index of P_k is
 *             L+1+k.  Digit j = chain limbs [j*alpha, min((j+1)*alpha, l+1)), alpha =
 *             ceil((L+1)/dnum), beta(l) = ceil((l+1)/alpha) (§2.1).
 *   Keys      evk layout [evk_digits][2][L+1+K][N]: evk[j][0] = b_j, evk[j][1] = a_j, EVAL.  Every call
 *             that reads a key takes the key's digit count `evk_digits`: the call needs the first
 *             beta(level) digits, so a key generated with fewer digits than the context's dnum is
 *             usable at the levels it covers.  evk_digits < beta(level) or > dnum -> HKS_EKEY
 *             ("ksk digit count < beta"), checked before any launch.  A key from
 *             hks_evk_prepare is passed with evk_digits | HKS_EVK_PREPARED.
 *   Streams   Every compute call is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *             legacy default stream).  Argument errors return synchronously before any launch;
 *             launch failures return HKS_ECUDA; asynchronous device faults surface on the
 *             caller's next synchronisation.
 *   Aliasing  In place is allowed only for hks_ntt_fwd / hks_ntt_inv.  All other outputs must not
 *             overlap inputs (HKS_EINVAL when detectable from pointer ranges).
 *   Errors    Status codes only; no exception crosses the ABI.  hks_last_error() returns a
 *             thread-local description of the last non-OK status on the calling thread.
 *   Threads   A context is immutable after creation and may be used concurrently from several
 *             host threads / streams, each with its own workspace.
 */
#ifndef HKS_H
#define HKS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hks_ctx hks_ctx;

typedef enum {
    HKS_OK = 0,
    HKS_EINVAL = 1,     /* bad argument: NULL, size, level > L, aliasing, nlimbs = 0 ... */
    HKS_ENOTPRIME = 2,  /* a modulus is not prime */
    HKS_ENOTNTT = 3,    /* a modulus is not 1 mod 2N */
    HKS_ERANGE = 4,     /* modulus >= 2^60, log_n outside [10, 17], dnum outside [1, L+1] */
    HKS_EDUP = 5,       /* a modulus appears twice in q || p */
    HKS_EKEY = 6,       /* evk_digits < beta(level) or > the context's dnum */
    HKS_EGALOIS = 7,    /* Galois element even or >= 2N */
    HKS_ECUDA = 8,      /* a CUDA runtime call or kernel launch failed */
    HKS_ENOMEM = 9,     /* device table allocation failed at context creation */
    HKS_EDEVICE = 10    /* host-only context (device < 0) used for compute, or wrong device */
} hks_status;

/* Operation selector for hks_workspace_bytes(). */
typedef enum {
    HKS_OP_MODUP = 0,           /* hks_modup */
    HKS_OP_MODDOWN = 1,         /* hks_moddown */
    HKS_OP_KEYSWITCH = 2,       /* hks_keyswitch */
    HKS_OP_ROTATE_HOISTED = 3,  /* hks_rotate_hoisted: count = the largest nrot of any call that will use
                                   the buffer (the layout has one accumulator region per concurrent
                                   branch); count = 0 returns the worst case over every nrot */
    HKS_OP_HMULT = 4,           /* hks_hmult */
    HKS_OP_RESCALE = 5          /* hks_rescale (count = npoly; 0 at level 0) */
} hks_op;

#define HKS_MAX_DIGITS 64

typedef struct hks_info {
    uint32_t log_n, n;          /* ring degree N = 2^log_n */
    uint32_t num_q, num_p;      /* L+1 and K */
    uint32_t dnum, alpha;       /* digits in the key, limbs per digit */
    uint32_t level, beta;       /* the queried level and its active digit count */
    uint32_t digit_lo[HKS_MAX_DIGITS], digit_hi[HKS_MAX_DIGITS];  /* digit j = [lo, hi) at `level` */
    int32_t device;             /* CUDA device ordinal, -1 for a host-only context */
} hks_info;

/* Thread-local text for the last non-OK status returned on this thread ("" if none). */
const char *hks_last_error(void);

/* Context creation (§3.5 precomputation; SPEC.md:297-305 create_context).
 *   log_n   10..17;  q[num_q] the chain q_0..q_L;  p[num_p] the special primes (K >= 1, any K:
 *           SURVEY.md §8(c) reading 15b);  dnum in [1, num_q].
 *   Every modulus must be prime, < 2^60, = 1 mod 2N, and all must be distinct.
 *   device  CUDA ordinal that will own the tables; -1 builds a host-only context that supports
 *           hks_ctx_query / hks_ctx_psi / hks_workspace_bytes only (compute calls: HKS_EDEVICE).
 *   *out    receives the context (owned by the caller, release with hks_ctx_destroy).
 * Builds, per prime: psi, forward/inverse twiddles with Shoup companions, N^-1; per (level,
 * digit): the Eq. 1 ModUp constants; the ModDown constants; then uploads them (device >= 0). */
hks_status hks_ctx_create(uint32_t log_n, const uint64_t *q, uint32_t num_q, const uint64_t *p,
                          uint32_t num_p, uint32_t dnum, int device, hks_ctx **out);

/* Releases the context and its device tables.  NULL is ignored.  No call may be in flight. */
void hks_ctx_destroy(hks_ctx *ctx);

/* Structural query at `level` (0..L): N, L+1, K, dnum, alpha, beta(level), digit ranges. */
hks_status hks_ctx_query(const hks_ctx *ctx, uint32_t level, hks_info *out);

/* psi of prime `prime_idx` (the minimal primitive 2N-th root; SURVEY.md §8(c) reading 1). */
hks_status hks_ctx_psi(const hks_ctx *ctx, uint32_t prime_idx, uint64_t *psi);

/* Bytes of device workspace `op` needs at `level` (0 if the op needs none). */
size_t hks_workspace_bytes(const hks_ctx *ctx, hks_op op, uint32_t level, uint32_t count);

/* Batched forward negacyclic NTT, in place (§3.6.4).
 *   x          [nlimbs][N] COEFF in, EVAL out (in place).
 *   prime_idx  host array [nlimbs]: limb b is reduced modulo prime prime_idx[b].
 * Output canonical.  Inputs must be canonical. */
hks_status hks_ntt_fwd(const hks_ctx *ctx, uint64_t *x, const uint32_t *prime_idx, uint32_t nlimbs,
                       void *stream);

/* Batched inverse NTT, in place, including N^-1 (§3.6.4). */
hks_status hks_ntt_inv(const hks_ctx *ctx, uint64_t *x, const uint32_t *prime_idx, uint32_t nlimbs,
                       void *stream);

/* Fast base conversion, Eq. 1 (§3.6.3):
 *   out_t = [ sum_i [x_i * qhat_i^-1]_{q_i} * [qhat_i]_t ]_t ,  qhat_i = prod_{m in src, m != i} m
 *   x       [nsrc][N] COEFF, limb i modulo prime src_idx[i];  out [ndst][N] COEFF.
 *   src_idx / dst_idx are host arrays of prime indices; nsrc <= 16, ndst <= 128, src and dst
 *   disjoint.  The result is the unique Eq. 1 value with canonical y_i (SURVEY.md reading 16).
 *   ws      hks_bconv_workspace_bytes(ctx, nsrc, ndst) bytes of device memory: the call derives this
 *           (src, dst) pair's Eq. 1 constants on the device into ws (no allocation, no host->device
 *           copy, graph-capturable), scales y_i = [x_i qhat_i^-1]_{q_i} into ws, then converts. */
hks_status hks_bconv(const hks_ctx *ctx, const uint64_t *x, const uint32_t *src_idx, uint32_t nsrc,
                     const uint32_t *dst_idx, uint32_t ndst, uint64_t *out, void *ws, void *stream);
size_t hks_bconv_workspace_bytes(const hks_ctx *ctx, uint32_t nsrc, uint32_t ndst);

/* ModUp (§3.6.3): digit decomposition + BConv + NTT.
 *   d    [l+1][N] EVAL at `level` = l.
 *   ext  [beta][l+1+K][N] EVAL: ext[j][t] = d[t] for t in digit j, otherwise
 *        NTT(BConv_{digit j -> t}(INTT(d[digit j]))).
 *   ws   hks_workspace_bytes(ctx, HKS_OP_MODUP, level, 0) bytes of device memory. */
hks_status hks_modup(const hks_ctx *ctx, const uint64_t *d, uint32_t level, uint64_t *ext, void *ws,
                     void *stream);

/* Evaluation-key inner product (§3.6.5 dot-product fusion):
 *   acc[0][t] = sum_{j<beta} D_j[t] * b_j[key(t)],  acc[1][t] = sum_j D_j[t] * a_j[key(t)]  (mod t)
 *   ext     [beta][l+1+K][N] EVAL (hks_modup output).  evk [evk_digits][2][L+1+K][N].
 *   galois  1 for none; otherwise odd k < 2N and D_j is replaced by its automorphism pi_k
 *           (EVAL permutation, hoisted order; SURVEY.md readings 14-15).
 *   acc     [2][l+1+K][N] EVAL. */
hks_status hks_ksk_inner_product(const hks_ctx *ctx, const uint64_t *ext, const uint64_t *evk,
                                 uint32_t evk_digits, uint32_t level, uint64_t galois, uint64_t *acc, void *stream);

/* ModDown (§3.6.5 "P^-1(x - NTT(x'))"):
 *   acc [l+1+K][N] EVAL -> out [l+1][N] EVAL,
 *   out_i = (acc_i - NTT(BConv_{P -> q_i}(INTT(acc_P)))_i) * P^-1 mod q_i.
 *   ws   hks_workspace_bytes(ctx, HKS_OP_MODDOWN, level, 0) bytes. */
hks_status hks_moddown(const hks_ctx *ctx, const uint64_t *acc, uint32_t level, uint64_t *out, void *ws,
                       void *stream);

/* Key preparation (optional, bit-exact by construction): evk_out = evk_in with every Q limb
 * (key limb index t <= L, both components of every digit) multiplied by [P^-1]_{q_t}; the P limbs are copied
 * unscaled.  Because acc = sum_j D_j evk_j is linear in the key, ModDown's (acc_Q - NTT(conv)) P^-1 becomes
 * acc'_Q - NTT(conv') with the P^-1 folded into the P -> Q conversion matrix (a context table): the
 * ModDown epilogue loses one modular product per output, and the outputs are identical in every Z_{q_i}.
 * Done once per key at load time; no Shoup companion is stored (it would double the key stream).
 *   evk_in, evk_out  [evk_digits][2][L+1+K][N] EVAL, 1 <= evk_digits <= dnum (else HKS_EKEY); evk_out ==
 *                    evk_in (in place) or disjoint (HKS_EINVAL on partial overlap); caller-owned.
 * The prepared key is passed to hks_keyswitch, hks_relinearize, hks_hmult, hks_rotate_hoisted,
 * hks_rotate_hoisted_batch and hks_linear_transform as evk_digits | HKS_EVK_PREPARED.  The step-level
 * hks_ksk_inner_product rejects it (HKS_EINVAL: hks_moddown would apply P^-1 twice), and so do the
 * limb-sharded hks_shard_* calls (HKS_EKEY). */
#define HKS_EVK_PREPARED 0x10000u
hks_status hks_evk_prepare(const hks_ctx *ctx, const uint64_t *evk_in, uint32_t evk_digits, uint64_t *evk_out,
                           void *stream);

/* Hybrid KeySwitch of ct = (c0, c1) at `level`:
 *   out0 = c0 + ModDown(acc0), out1 = ModDown(acc1), acc = KIP(ModUp(c1), evk).
 *   Relinearisation of (d0, d1, d2): call with (c0, c1) = (0-or-d0, d2) and add d1 to out1.
 *   c0 may be NULL (then out0 = ModDown(acc0)).  c0, c1, out0, out1: [l+1][N] EVAL.
 *   evk [evk_digits][2][L+1+K][N], beta(level) <= evk_digits <= dnum (else HKS_EKEY).
 *   ws   hks_workspace_bytes(ctx, HKS_OP_KEYSWITCH, level, 0) bytes. */
hks_status hks_keyswitch(const hks_ctx *ctx, const uint64_t *c0, const uint64_t *c1, uint32_t level,
                         const uint64_t *evk, uint32_t evk_digits, uint64_t *out0, uint64_t *out1, void *ws,
                         void *stream);

/* Relinearisation of a tensor-product ciphertext (d0, d1, d2) at `level` (HMult's KeySwitch,
 * PAPER.md:75 Table 1 HMult, PAPER.md:351 HMult fusion):  out0 = d0 + ModDown(acc0),
 * out1 = d1 + ModDown(acc1), acc = KIP(ModUp(d2), evk).  Both additions are fused in the ModDown
 * epilogue.  d0 may be NULL (treated as 0); d1 must not be NULL.  Layouts and ws as hks_keyswitch. */
hks_status hks_relinearize(const hks_ctx *ctx, const uint64_t *d0, const uint64_t *d1, const uint64_t *d2,
                           uint32_t level, const uint64_t *evk, uint32_t evk_digits, uint64_t *out0, uint64_t *out1,
                           void *ws,
                           void *stream);

/* HMult without rescale (Table 1 "HMult"; §3.6.5 HMult fusion; DESIGN.md
 * reading 16) of ct_a = (a0, a1) and ct_b = (b0, b1) at `level`, all [l+1][N] EVAL canonical:
 *   d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 (mod q_i);
 *   out0 = d0 + ModDown(acc0), out1 = d1 + ModDown(acc1), acc = KIP(ModUp(d2), evk)  (evk = relin key).
 * Fused: d2 is formed inside the first INTT pass, d0 / d1 inside the ModDown epilogue.  Outputs must
 * not overlap any input or ws.  ws: hks_workspace_bytes(ctx, HKS_OP_HMULT, level, 0) bytes. */
hks_status hks_hmult(const hks_ctx *ctx, const uint64_t *a0, const uint64_t *a1, const uint64_t *b0,
                     const uint64_t *b1, uint32_t level, const uint64_t *evk, uint32_t evk_digits, uint64_t *out0,
                     uint64_t *out1,
                     void *ws, void *stream);

/* Rescale of npoly polynomials from level l >= 1 to l - 1 (Table 1 "Rescale after
 * multiplication"; §3.6.5 "q_l^{-1}(x^(i) - NTT(SwitchModulo(x^(l))))"; DESIGN.md reading
 * 15: centered SwitchModulo, i.e. the CRT value of the output is round(X / q_l)):
 *   x   [npoly][l+1][N] EVAL canonical;  out [npoly][l][N] EVAL canonical (polynomial p at p*l*N).
 *   A ciphertext is npoly = 2 (c0, c1 contiguous).  HKS_EINVAL at level 0, on overlap, NULL.
 *   ws: hks_workspace_bytes(ctx, HKS_OP_RESCALE, level, npoly) bytes. */
hks_status hks_rescale(const hks_ctx *ctx, const uint64_t *x, uint32_t npoly, uint32_t level, uint64_t *out,
                       void *ws, void *stream);

/* Fused plaintext-weighted sum of ciphertexts (§3.6.5 "a weighed sum can be reduced from
 * 4n-2 down to n+1 memory operations"):  out_p = sum_{j<nterm} w[j] * x_p[j]  (mod q_i), p = 0, 1.
 *   w[j], x0[j], x1[j]: host arrays of nterm device pointers, each [l+1][N] EVAL canonical (w[j] a
 *   plaintext, (x0[j], x1[j]) a ciphertext); out0, out1 [l+1][N] EVAL canonical, must not overlap any
 *   term.  One 128-bit accumulation and one reduction per output (16 terms per pass). */
hks_status hks_pt_weighted_sum(const hks_ctx *ctx, uint32_t nterm, const uint64_t *const *w,
                               const uint64_t *const *x0, const uint64_t *const *x1, uint32_t level,
                               uint64_t *out0, uint64_t *out1, void *stream);

/* Ciphertext x plaintext-matrix product by baby-step giant-step (§3.6.7: "performed using
 * a BSGS algorithm ... leverages the hoisted rotation optimization"; no ModDown hoisting):
 *   ct_0 = (c0, c1);  ct_j = RotHoisted(ct, baby_galois[j-1], baby_evk[j-1]), j = 1..n1-1 (one ModUp);
 *   I_i = sum_j pt[i*n1 + j] * ct_j   (hks_pt_weighted_sum);
 *   out = I_0 + sum_{i=1..n2-1} RotHoisted(I_i, giant_galois[i-1], giant_evk[i-1]).
 *   pt: host array of n1*n2 device pointers to the (pre-rotated) diagonals [l+1][N] EVAL; galois / evk:
 *   host arrays (n1-1 and n2-1 entries).  out0/out1 [l+1][N] must not overlap the inputs or ws.
 *   ws: hks_linear_transform_workspace_bytes(ctx, level, n1) bytes.
 *   Stream semantics: with n2 > 2 the independent giant steps are spread round-robin over `stream` and
 *   the context's three side streams (forked from `stream` by an event, joined back before the last
 *   accumulation), so the whole call stays ordered on `stream` and can be captured into a CUDA graph. */
hks_status hks_linear_transform(const hks_ctx *ctx, const uint64_t *c0, const uint64_t *c1, uint32_t level,
                                uint32_t n1, uint32_t n2, const uint64_t *baby_galois,
                                const uint64_t *const *baby_evk, const uint64_t *giant_galois,
                                const uint64_t *const *giant_evk, uint32_t evk_digits, const uint64_t *const *pt,
                                uint64_t *out0,
                                uint64_t *out1, void *ws, void *stream);
size_t hks_linear_transform_workspace_bytes(const hks_ctx *ctx, uint32_t level, uint32_t n1);

/* EVAL-form automorphism X -> X^galois on nlimbs limbs (prime-independent permutation,
 * SPEC.md:244-252; SURVEY.md reading 15):  out[l][j] = in[l][j'], 2brv(j')+1 = k(2brv(j)+1) mod 2N.
 * in != out required. */
hks_status hks_automorph(const hks_ctx *ctx, const uint64_t *in, uint32_t nlimbs, uint64_t galois,
                         uint64_t *out, void *stream);

/* Hoisted rotations (§3.6.6): one ModUp of c1 shared by nrot rotations.
 *   galois[r], evk[r], out0[r], out1[r]: host arrays of length nrot (device pointers inside).
 *   out0[r] = pi_k(c0) + ModDown(acc0_r), out1[r] = ModDown(acc1_r), acc_r = KIP(ext, evk[r], k_r).
 *   ws   hks_workspace_bytes(ctx, HKS_OP_ROTATE_HOISTED, level, nrot) bytes.
 *   Stream semantics: with nrot > 1 the rotations after the shared ModUp are split over `stream` and the
 *   context's three side streams (event fork / join); the call stays ordered on `stream`, graph-capturable. */
hks_status hks_rotate_hoisted(const hks_ctx *ctx, const uint64_t *c0, const uint64_t *c1, uint32_t level,
                              uint32_t nrot, const uint64_t *galois, const uint64_t *const *evk, uint32_t evk_digits,
                              uint64_t *const *out0, uint64_t *const *out1, void *ws, void *stream);


/* Hoisted rotations of nct <= 8 ciphertexts sharing the same nrot rotation keys (SURVEY.md §7 "key
 * streaming": the key product loads every key word once for the whole batch).  c0[i], c1[i]:
 * ciphertext i [l+1][N] EVAL; out0/out1[i * nrot + r] receive rotation r of ciphertext i (as in
 * hks_rotate_hoisted).  beta(level) <= 4.  ws: hks_rotate_hoisted_batch_workspace_bytes(ctx, nct, level).
 * Stream semantics: after the ModUps the nrot rotations are spread round-robin over `stream` and the
 * context's three side streams (event fork / join), so the call stays ordered on `stream` and is graph-capturable. */
hks_status hks_rotate_hoisted_batch(const hks_ctx *ctx, uint32_t nct, const uint64_t *const *c0,
                                    const uint64_t *const *c1, uint32_t level, uint32_t nrot,
                                    const uint64_t *galois, const uint64_t *const *evk, uint32_t evk_digits,
                                    uint64_t *const *out0,
                                    uint64_t *const *out1, void *ws, void *stream);
size_t hks_rotate_hoisted_batch_workspace_bytes(const hks_ctx *ctx, uint32_t nct, uint32_t level);

/* ---- diagnostics (bench.py evidence; not part of the key-switching math) ---------------------
 * hks_launch_count: number of kernels this library has launched in this process (all contexts).
 * hks_prof_enable(1): from now on every kernel launch is bracketed by a CUDA event pair recorded on
 *   the launch's stream, tagged with its kernel class and its algorithmic bytes (limb words read and
 *   written, excluding twiddle/constant tables).  hks_prof_enable(0) stops recording.
 * hks_prof_read: synchronises the recorded events and returns, per kernel class, the launch count,
 *   the summed device time (ms), algorithmic bytes and algorithmic multiplies; clears the record.  Returns the
 *   number of classes written (<= max). */
typedef struct hks_prof_entry {
    char name[32];
    uint64_t launches;
    double total_ms;
    double bytes;   /* algorithmic HBM bytes (limb words read + written) */
    double muls;    /* algorithmic 32x32->64-bit integer partial products (4 per exact 60x60-bit
                       product; 7 wide-equivalents per Shoup butterfly) */
} hks_prof_entry;

uint64_t hks_launch_count(void);
hks_status hks_prof_enable(int on);
int hks_prof_read(hks_prof_entry *out, int max);

/* ---- limb-sharded KeySwitch (BASELINE.json configs[3]) ------------------
 * `world` ranks (one per GPU) each own a contiguous, balanced slice of the chain limbs q_0..q_L and
 * of the special limbs p_0..p_{K-1} (the paper's LimbPartition, §3.3, which the paper
 * leaves "in development").  Base conversion needs every source limb of a coefficient, so a
 * KeySwitch is three local phases around two all-gathers that the caller issues (NCCL over NVLink,
 * torch.distributed.all_gather_into_tensor) on the same stream:
 *   A  hks_shard_ks_modup_in    : ysend = INTT(c1_loc) * N^-1 [qhat]^-1          (COEFF, owned chain limbs)
 *      all-gather #1            : yall[world][q_pad][N] <- ysend[q_pad][N]
 *   B  hks_shard_ks_inner       : BConv to owned limbs + NTT + key inner product -> acc_loc;
 *                                 ypsend = INTT(acc_loc[P]) * N^-1 [phat]^-1      (owned special limbs)
 *      all-gather #2            : ypall[world][2][p_pad][N] <- ypsend[2][p_pad][N]
 *   C  hks_shard_ks_moddown_out : BConv P -> owned chain limbs + NTT + (acc - .) P^-1 (+ c0)
 * The result is bit-identical to hks_keyswitch restricted to the owned limbs.
 * Local layouts: c0_loc, c1_loc, out0_loc, out1_loc [nq_act][N] (owned chain limbs <= level, in
 * order); evk_loc [evk_digits][2][nkey][N] (owned chain limbs of the full chain, then owned special limbs);
 * acc_loc [2][nq_act + (p_hi - p_lo)][N]. */
typedef struct hks_shard_info {
    uint32_t world, rank, level;
    uint32_t q_lo, q_hi;     /* owned chain limbs [q_lo, q_hi) of q_0..q_L */
    uint32_t p_lo, p_hi;     /* owned special limbs [p_lo, p_hi) of p_0..p_{K-1} */
    uint32_t nq_act;         /* owned chain limbs active at `level` */
    uint32_t q_pad, p_pad;   /* all-gather chunk sizes (limbs): max owned chain / special limbs */
    uint32_t nkey;           /* owned key limbs = (q_hi - q_lo) + (p_hi - p_lo) */
} hks_shard_info;

hks_status hks_shard_query(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank, hks_shard_info *out);
size_t hks_shard_workspace_bytes(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank);
hks_status hks_shard_ks_modup_in(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                 const uint64_t *c1_loc, uint64_t *ysend, void *stream);
hks_status hks_shard_ks_inner(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                              const uint64_t *yall, const uint64_t *c1_loc, const uint64_t *evk_loc, uint32_t evk_digits,
                              uint64_t *acc_loc, uint64_t *ypsend, void *ws, void *stream);
hks_status hks_shard_ks_moddown_out(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                    const uint64_t *ypall, const uint64_t *acc_loc, const uint64_t *c0_loc,
                                    uint64_t *out0_loc, uint64_t *out1_loc, void *ws, void *stream);

/* Pipelined phase B (SURVEY.md §8(f) NEXT-3 "per-digit pipelined all-gather overlapped with BConv"): the
 * same work and result as hks_shard_ks_inner, but the base conversion of digit j is enqueued only after
 * `stream` waits on digit_ready[j] -- a HOST array of beta(level) cudaEvent_t handles (as void*; an entry may
 * be NULL for a digit already delivered) -- so the caller can deliver yall digit by digit (e.g. one NCCL
 * broadcast per (digit, owner) segment, shard.PipelinedShardedKeySwitch) and the conversion of digit j overlaps
 * the transfer of digit j + 1.  yall is read only at the slots of each digit's limbs, in the layout of
 * hks_shard_ks_inner (rank r's limbs at [r * q_pad, r * q_pad + q_hi - q_lo)). */
hks_status hks_shard_ks_inner_pipelined(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                        const uint64_t *yall, const void *const *digit_ready, const uint64_t *c1_loc,
                                        const uint64_t *evk_loc, uint32_t evk_digits, uint64_t *acc_loc,
                                        uint64_t *ypsend, void *ws, void *stream);

/* Peer-memory variants of phases B and C (the collective fused into the base
 * conversion over NVLink).  Instead of an all-gathered buffer, the caller passes a HOST array of `world`
 * device pointers: rank r's ysend ([q_pad][N]) resp. ypsend ([2][p_pad][N]) as mapped into this rank's
 * address space (its own buffer for r == rank; a peer mapping -- CUDA IPC / symmetric memory over
 * NVLink -- for the others; plain device pointers when several simulated ranks share one GPU).  The
 * base-conversion kernel loads every source limb directly from its owner, so no all-gather runs and
 * each rank reads only the limbs its targets need.  Same outputs as the all-gather phases, bit for bit.
 * Ordering is the caller's: every rank's phase A (resp. B) must be complete and visible before any rank
 * starts phase B (resp. C), and no rank may overwrite its ysend / ypsend until all peers finished
 * reading it (e.g. a symmetric-memory barrier on the stream).  Errors: HKS_EINVAL for a NULL table or
 * entry, plus those of the all-gather phases. */
hks_status hks_shard_ks_inner_peer(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                   const uint64_t *const *ysend_ranks, const uint64_t *c1_loc,
                                   const uint64_t *evk_loc, uint32_t evk_digits, uint64_t *acc_loc, uint64_t *ypsend, void *ws,
                                   void *stream);
hks_status hks_shard_ks_moddown_out_peer(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                         const uint64_t *const *ypsend_ranks, const uint64_t *acc_loc,
                                         const uint64_t *c0_loc, uint64_t *out0_loc, uint64_t *out1_loc, void *ws,
                                         void *stream);

/* All-to-all coefficient-sharded KeySwitch (SURVEY.md §8(e) "coefficient-sharded BConv", §8(f) NEXT-3;
 * PAPER.md:219 LimbPartition).  Same limb ownership as the phases above, but the base
 * conversions work on a coefficient chunk of every limb instead of every coefficient of the owned limbs:
 * rank k's chunk is rows [k R / G, (k + 1) R / G) of the R x C limb layout (N = R C, G = world, a power of two
 * <= R), Nc = N / G words per limb.  A buffer "[G][S][Nc]" is coefficient-chunked: chunk k of slot s at
 * (k S + s) Nc -- the input / output of torch.distributed.all_to_all_single, which sends part k to rank k.
 * Five local phases around four all-to-alls the caller issues on the same stream:
 *   1  hks_shard_a2a_modup_in      ysend [G][q_pad][Nc] = chunks of INTT(c1_loc) N^-1 [qhat]^-1
 *      all-to-all #1               yrecv [G][q_pad][Nc]: rank r's active chain limbs, this rank's chunk
 *   2  hks_shard_a2a_bconv         extsend [G][beta][n_pad][Nc]: Eq. 1 of every digit on this chunk to every
 *                                  extended limb outside the digit, part d holding rank d's owned targets
 *                                  (slot j n_pad + u, u = index in d's list: active chain limbs, then P limbs)
 *      all-to-all #2               extrecv [G][beta][n_pad][Nc]: chunk r of this rank's converted limbs
 *   3  hks_shard_a2a_inner         NTT + key inner product -> acc_loc (as hks_shard_ks_inner); ypsend
 *                                  [G][2][p_pad][Nc] = chunks of INTT(acc_loc[P]) N^-1 [phat]^-1
 *      all-to-all #3               yprecv [G][2][p_pad][Nc]
 *   4  hks_shard_a2a_moddown_bconv convsend [G][2][nq_pad][Nc]: Eq. 1 P -> every active chain limb on this chunk,
 *                                  part d holding rank d's limbs (slot p nq_pad + i - q_lo(d))
 *      all-to-all #4               convrecv [G][2][nq_pad][Nc]
 *   5  hks_shard_a2a_moddown_out   out_p = (acc_p - NTT(conv_p)) P^-1 (+ c0) on the owned active chain limbs
 * Per-rank receive volume: the source chunks of all limbs plus the owned converted limbs, instead of every
 * chain / special limb whole (all-gather).  Bit-identical to hks_keyswitch on the owned limbs.  Pad slots are
 * never read.  ws: hks_shard_a2a_workspace_bytes.  Layouts c0/c1/out/evk/acc as the all-gather phases. */
typedef struct hks_shard_a2a_info {
    uint32_t chunk_words;   /* Nc = N / world */
    uint32_t n_pad;         /* max owned extended limbs (active chain + special) over the ranks */
    uint32_t nq_pad;        /* max owned active chain limbs over the ranks */
    uint32_t beta;          /* digits at the level */
} hks_shard_a2a_info;

hks_status hks_shard_a2a_query(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                               hks_shard_a2a_info *out);
size_t hks_shard_a2a_workspace_bytes(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank);
hks_status hks_shard_a2a_modup_in(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                  const uint64_t *c1_loc, uint64_t *ysend, void *ws, void *stream);
hks_status hks_shard_a2a_bconv(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                               const uint64_t *yrecv, uint64_t *extsend, void *stream);
hks_status hks_shard_a2a_inner(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                               const uint64_t *extrecv, const uint64_t *c1_loc, const uint64_t *evk_loc,
                               uint32_t evk_digits, uint64_t *acc_loc, uint64_t *ypsend, void *ws, void *stream);
hks_status hks_shard_a2a_moddown_bconv(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                       const uint64_t *yprecv, uint64_t *convsend, void *stream);
hks_status hks_shard_a2a_moddown_out(const hks_ctx *ctx, uint32_t level, uint32_t world, uint32_t rank,
                                     const uint64_t *convrecv, const uint64_t *acc_loc, const uint64_t *c0_loc,
                                     uint64_t *out0_loc, uint64_t *out1_loc, void *ws, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HKS_H */
