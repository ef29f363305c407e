// shard.cu -- limb-sharded KeySwitch phases (include/hks.h "limb-sharded KeySwitch").
//
// Ownership (full index space, independent of the level so keys are distributed once): chain limbs
// q_0..q_L in `world` contiguous chunks, the first (L+1) mod world ranks one limb larger; special
// limbs p_0..p_{K-1} in contiguous chunks, the LAST K mod world ranks one limb larger (they own fewer
// chain limbs).  Every step reuses the single-GPU kernels with slot maps into the gathered buffers.
#include <algorithm>

#include "internal.h"

namespace {

struct Plan {
    u32 world, rank, level;
    u32 q_lo, q_hi, p_lo, p_hi, nq_act, q_pad, p_pad, nkey, np_own, n_own;
    std::vector<u32> qlo_r, qhi_r, plo_r, phi_r;   // per rank
    u32 q_owner(u32 i) const { for (u32 r = 0; r < world; r++) if (i < qhi_r[r]) return r; return world - 1; }
    u32 p_owner(u32 k) const { for (u32 r = 0; r < world; r++) if (k < phi_r[r]) return r; return world - 1; }
};

void chunks(u32 total, u32 world, bool extra_last, std::vector<u32> &lo, std::vector<u32> &hi) {
    lo.resize(world);
    hi.resize(world);
    const u32 base = total / world, rem = total % world;
    u32 at = 0;
    for (u32 r = 0; r < world; r++) {
        const bool extra = extra_last ? (r >= world - rem) : (r < rem);
        lo[r] = at;
        at += base + (extra ? 1 : 0);
        hi[r] = at;
    }
}

hks_status make_plan(const hks_ctx *c, u32 level, u32 world, u32 rank, Plan &P) {
    if (!c) HKS_FAIL(HKS_EINVAL, "shard: NULL context");
    if (world < 1 || rank >= world) HKS_FAIL(HKS_EINVAL, "shard: rank %u / world %u", rank, world);
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "shard: level %u > L", level);
    if (world > c->nq) HKS_FAIL(HKS_EINVAL, "shard: world %u larger than the chain", world);
    P.world = world; P.rank = rank; P.level = level;
    chunks(c->nq, world, false, P.qlo_r, P.qhi_r);
    chunks(c->np, world, true, P.plo_r, P.phi_r);
    P.q_lo = P.qlo_r[rank]; P.q_hi = P.qhi_r[rank];
    P.p_lo = P.plo_r[rank]; P.p_hi = P.phi_r[rank];
    P.nq_act = P.q_lo >= level + 1 ? 0 : std::min(P.q_hi, level + 1) - P.q_lo;
    P.q_pad = P.p_pad = 0;
    for (u32 r = 0; r < world; r++) {
        P.q_pad = std::max(P.q_pad, P.qhi_r[r] - P.qlo_r[r]);
        P.p_pad = std::max(P.p_pad, P.phi_r[r] - P.plo_r[r]);
    }
    P.np_own = P.p_hi - P.p_lo;
    P.nkey = (P.q_hi - P.q_lo) + P.np_own;
    P.n_own = P.nq_act + P.np_own;
    return HKS_OK;
}

hks_status dev_ctx(const hks_ctx *c) {
    if (c->device < 0) HKS_FAIL(HKS_EDEVICE, "host-only context cannot run device operations");
    return HKS_OK;
}

// BConv launch helper (same as capi.cu's, kept local)
hks_status bconv_groups(const hks_ctx *c, std::vector<BconvGroup> &groups, const u64 *in, u64 *out, cudaStream_t s) {
    size_t i = 0;
    while (i < groups.size()) {
        BconvArgs a{};
        a.in = in;
        a.out = out;
        a.pc = c->d_pc;
        a.log_n = c->log_n;
        a.lazy_out = 1;
        a.big = c->all_big ? 1 : 0;
        u32 ns = groups[i].nsrc, k = 0;
        while (i < groups.size() && k < BC_MAXG && groups[i].nsrc == ns) a.g[k++] = groups[i++];
        a.ngroups = k;
        hks_status st = launch_bconv(a, BC_MAXDST, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}

void push_group(std::vector<BconvGroup> &out, u32 nsrc, const u16 *src_slot, const uint2 *mat, u32 stride,
                const std::vector<u16> &ds, const std::vector<u16> &dp, const double *matf, const u32 *mats, const u64 *matb, const u64 *mimg,
                const u64 *const *srcp = nullptr) {
    for (size_t u0 = 0; u0 < ds.size(); u0 += BC_MAXDST) {
        BconvGroup g{};
        g.nsrc = nsrc;
        g.ndst = (u32)std::min<size_t>(BC_MAXDST, ds.size() - u0);
        g.mat_stride = stride;
        g.mat = mat + u0;
        g.matf = matf ? matf + 3 * u0 : nullptr;   // NULL unless HKS_EXPERIMENTAL uploaded the table
        g.mats = mats ? mats + u0 : nullptr;
        g.matb = matb ? matb + 8 * u0 : nullptr;
        g.mimg = mimg ? mimg + (size_t)bconv_img_words(nsrc) * u0 : nullptr;
        for (u32 i = 0; i < nsrc; i++) {
            g.src_slot[i] = src_slot[i];
            g.srcp[i] = srcp ? srcp[i] : nullptr;
        }
        for (u32 u = 0; u < g.ndst; u++) { g.dst_slot[u] = ds[u0 + u]; g.dst_prime[u] = dp[u0 + u]; }
        out.push_back(g);
    }
}

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) { cudaGetDevice(&prev); if (prev != dev) cudaSetDevice(dev); else prev = -1; }
    ~DevGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

}  // namespace

extern "C" hks_status hks_shard_query(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank, hks_shard_info *out) {
    if (!out) HKS_FAIL(HKS_EINVAL, "shard_query: NULL out");
    Plan P;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK) return st;
    *out = hks_shard_info{P.world, P.rank, P.level, P.q_lo, P.q_hi, P.p_lo, P.p_hi, P.nq_act, P.q_pad, P.p_pad, P.nkey};
    return HKS_OK;
}

extern "C" size_t hks_shard_workspace_bytes(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank) {
    Plan P;
    if (make_plan(c, level, world, rank, P) != HKS_OK) return 0;
    return ((size_t)c->beta(level) * P.n_own + 2 * (size_t)P.nq_act) * c->n * sizeof(u64);
}

// Phase A: ysend[li] = INTT(c1_loc[li]) * N^-1 [qhat_{j,i}]^-1, i = q_lo + li (canonical COEFF).
extern "C" hks_status hks_shard_ks_modup_in(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                           const uint64_t *c1_loc, uint64_t *ysend, void *stream) {
    Plan P;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if (P.nq_act == 0) return HKS_OK;
    if (!c1_loc || !ysend) HKS_FAIL(HKS_EINVAL, "shard_ks_modup_in: NULL buffer");
    DevGuard g(c->device);
    LimbList L;
    for (u32 li = 0; li < P.nq_act; li++) L.push(li, li, P.q_lo + li);
    return run_ntt(c, NTT_INV, L, c1_loc, ysend, c->d_mu_scale + c->mu_scale_off[level] + P.q_lo, P.nq_act,
                   (cudaStream_t)stream);
}

// Phase B: D_j for owned limbs from the gathered y, fused NTT + key inner product, then
// ypsend[p][kk] = INTT(acc_p[owned P_kk]) * N^-1 [phat_k]^-1.
// yall != NULL: sources are slots of the all-gathered buffer; else peers[r] is rank r's ysend (a local or
// peer-mapped device address) and the base conversion reads every source limb straight from its owner.
// digit_ready != NULL (pipelined phase B): the stream waits on digit_ready[j] before the base conversion of
// digit j, one conversion launch per digit.
static hks_status shard_inner(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank, const uint64_t *yall,
                              const uint64_t *const *peers, const uint64_t *c1_loc, const uint64_t *evk_loc,
                              uint32_t evk_digits, uint64_t *acc_loc, uint64_t *ypsend, void *ws, void *stream,
                              const void *const *digit_ready = nullptr) {
    Plan P;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if ((!yall && !peers) || !evk_loc || !acc_loc || !ypsend || !ws || (P.nq_act && !c1_loc))
        HKS_FAIL(HKS_EINVAL, "shard_ks_inner: NULL buffer");
    if (peers)
        for (u32 r = 0; r < world; r++)
            if (!peers[r]) HKS_FAIL(HKS_EINVAL, "shard_ks_inner_peer: NULL buffer of rank %u", r);
    const u32 beta = c->beta(level), ne = c->ne(level);
    if (beta > FK_MAXD) HKS_FAIL(HKS_EINVAL, "shard_ks_inner: beta %u > %d", beta, FK_MAXD);
    if (evk_digits < beta || evk_digits > c->dnum)
        HKS_FAIL(HKS_EKEY, "shard_ks_inner: key has %u digits; level %u needs %u (context dnum %u)", evk_digits, level,
                 beta, c->dnum);
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    u64 *ext = (u64 *)ws;
    // owned extended limbs: chain t in [q_lo, q_lo + nq_act), then special P_k, k in [p_lo, p_hi)
    std::vector<u32> own_t;
    for (u32 li = 0; li < P.nq_act; li++) own_t.push_back(P.q_lo + li);
    for (u32 k = P.p_lo; k < P.p_hi; k++) own_t.push_back(level + 1 + k);
    // BConv per digit to the owned targets outside the digit; matrix columns of (level, digit) follow
    // the target order t in [0, ne) \ digit, so owned targets map to column positions.
    std::vector<BconvGroup> groups;
    std::vector<size_t> gfirst;   // first group of digit j
    LimbList T;
    for (u32 j = 0; j < beta; j++) {
        gfirst.push_back(groups.size());
        const u32 lo = c->digit_lo(j), hi = c->digit_hi(level, j);
        u16 src[BC_MAXSRC];
        const u64 *srcp[BC_MAXSRC];
        for (u32 i = lo; i < hi; i++) {
            const u32 r = P.q_owner(i);
            src[i - lo] = (u16)(r * P.q_pad + (i - P.qlo_r[r]));
            srcp[i - lo] = peers ? peers[r] + (size_t)(i - P.qlo_r[r]) * c->n : nullptr;
        }
        const size_t moff = c->mu_mat_off[(size_t)level * c->dnum + j];
        const uint2 *mat = c->d_mu_mat + moff;
        const double *matf = tab_at(c->d_mu_matf, 3 * moff);
        const u32 *mats = c->d_mu_mats + moff;
        const u64 *matb = tab_at(c->d_mu_matb, 8 * moff);
        const u64 *mimg = c->d_mu_img + c->mu_img_off[(size_t)level * c->dnum + j];
        const u32 imgw = bconv_img_words(hi - lo);
        const u32 ntg = ne - (hi - lo);
        // contiguous runs of column positions
        std::vector<u16> ds, dp;
        int run_col = -1;
        auto flush = [&]() {
            if (!ds.empty()) push_group(groups, hi - lo, src, mat + run_col, ntg, ds, dp, tab_at(matf, 3 * run_col), mats + run_col,
                                         tab_at(matb, 8 * run_col), mimg + (size_t)imgw * run_col, srcp);
            ds.clear(); dp.clear(); run_col = -1;
        };
        int prev_col = -2;
        for (u32 u = 0; u < own_t.size(); u++) {
            const u32 t = own_t[u];
            if (t >= lo && t < hi) continue;
            const int col = (int)(t < lo ? t : t - (hi - lo));
            if (col != prev_col + 1) { flush(); run_col = col; }
            ds.push_back((u16)(j * P.n_own + u));
            dp.push_back((u16)c->ext_prime(level, t));
            T.push(j * P.n_own + u, j * P.n_own + u, c->ext_prime(level, t));
            prev_col = col;
        }
        flush();
    }
    gfirst.push_back(groups.size());
    if (!digit_ready) {
        if ((st = bconv_groups(c, groups, yall ? yall : ext, ext, s)) != HKS_OK) return st;
    } else {
        for (u32 j = 0; j < beta; j++) {
            if (digit_ready[j] && cudaStreamWaitEvent(s, (cudaEvent_t)digit_ready[j], 0) != cudaSuccess)
                HKS_FAIL(HKS_ECUDA, "shard_ks_inner_pipelined: wait on digit %u", j);
            std::vector<BconvGroup> gj(groups.begin() + gfirst[j], groups.begin() + gfirst[j + 1]);
            if (!gj.empty() && (st = bconv_groups(c, gj, yall, ext, s)) != HKS_OK) return st;
        }
    }
    if (T.size() && (st = run_ntt_fwd_cols(c, T, ext, ext, s)) != HKS_OK) return st;
    std::vector<KipItem> items(own_t.size());
    for (u32 u = 0; u < own_t.size(); u++) {
        const u32 t = own_t[u];
        KipItem &it = items[u];
        it.prime = (u16)c->ext_prime(level, t);
        it.kslot = (u16)(t <= level ? t - P.q_lo : (P.q_hi - P.q_lo) + (t - level - 1 - P.p_lo));
        it.aslot = (u16)u;
        for (u32 j = 0; j < beta; j++) {
            const bool own = t <= level && t >= c->digit_lo(j) && t < c->digit_hi(level, j);
            it.src[j] = own ? (u16)(FK_DIRECT | (t - P.q_lo)) : (u16)(j * P.n_own + u);
        }
    }
    if ((st = run_ntt_kip(c, items, beta, ext, c1_loc, evk_loc, acc_loc, P.nkey, P.n_own, s)) != HKS_OK) return st;
    if (P.np_own) {
        LimbList L;
        for (u32 p = 0; p < 2; p++)
            for (u32 kk = 0; kk < P.np_own; kk++) L.push(p * P.n_own + P.nq_act + kk, p * P.p_pad + kk, c->nq + P.p_lo + kk);
        // scale index b % np_own = kk
        if ((st = run_ntt(c, NTT_INV, L, acc_loc, ypsend, c->d_md_scale + P.p_lo, P.np_own, s)) != HKS_OK) return st;
    }
    return HKS_OK;
}

// Phase C: conv_p = BConv_{P -> owned chain}(ypall_p); out_p = (acc_p - NTT(conv_p)) P^-1 (+ c0 on p = 0).
static hks_status shard_moddown(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank, const uint64_t *ypall,
                                const uint64_t *const *peers, const uint64_t *acc_loc, const uint64_t *c0_loc,
                                uint64_t *out0_loc, uint64_t *out1_loc, void *ws, void *stream) {
    Plan P;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if (P.nq_act == 0) return HKS_OK;
    if ((!ypall && !peers) || !acc_loc || !out0_loc || !out1_loc || !ws)
        HKS_FAIL(HKS_EINVAL, "shard_ks_moddown_out: NULL buffer");
    if (peers)
        for (u32 r = 0; r < world; r++)
            if (!peers[r]) HKS_FAIL(HKS_EINVAL, "shard_ks_moddown_out_peer: NULL buffer of rank %u", r);
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const u32 beta = c->beta(level), K = c->np;
    u64 *conv = (u64 *)ws + (size_t)beta * P.n_own * c->n;
    std::vector<BconvGroup> groups;
    for (u32 p = 0; p < 2; p++) {
        u16 src[BC_MAXSRC];
        const u64 *srcp[BC_MAXSRC];
        for (u32 k = 0; k < K; k++) {
            const u32 r = P.p_owner(k);
            src[k] = (u16)(r * 2 * P.p_pad + p * P.p_pad + (k - P.plo_r[r]));
            srcp[k] = peers ? peers[r] + (size_t)(p * P.p_pad + (k - P.plo_r[r])) * c->n : nullptr;
        }
        std::vector<u16> ds(P.nq_act), dp(P.nq_act);
        for (u32 li = 0; li < P.nq_act; li++) { ds[li] = (u16)(p * P.nq_act + li); dp[li] = (u16)(P.q_lo + li); }
        push_group(groups, K, src, c->d_md_mat + P.q_lo, c->nq, ds, dp, tab_at(c->d_md_matf, 3 * P.q_lo), c->d_md_mats + P.q_lo,
                   tab_at(c->d_md_matb, 8 * P.q_lo), c->d_md_img + (size_t)bconv_img_words(K) * P.q_lo, srcp);
    }
    if ((st = bconv_groups(c, groups, ypall ? ypall : conv, conv, s)) != HKS_OK) return st;
    LimbList M;
    std::vector<uint8_t> poly;
    for (u32 p = 0; p < 2; p++)
        for (u32 li = 0; li < P.nq_act; li++) {
            M.push(p * P.nq_act + li, li, P.q_lo + li, p * P.n_own + li, (p == 0 && c0_loc) ? li : 0xffff);
            poly.push_back((uint8_t)p);
        }
    std::vector<MdOut> mo = {MdOut{out0_loc, c0_loc, 1}, MdOut{out1_loc, nullptr, 1}};
    if ((st = run_ntt_moddown(c, M, poly, mo, conv, acc_loc, s)) != HKS_OK) return st;
    return HKS_OK;
}

extern "C" hks_status hks_shard_ks_inner(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                        const uint64_t *yall, const uint64_t *c1_loc, const uint64_t *evk_loc,
                                        uint32_t evk_digits, uint64_t *acc_loc, uint64_t *ypsend, void *ws,
                                        void *stream) {
    if (!yall) HKS_FAIL(HKS_EINVAL, "shard_ks_inner: NULL yall");
    return shard_inner(c, level, world, rank, yall, nullptr, c1_loc, evk_loc, evk_digits, acc_loc, ypsend, ws, stream);
}

extern "C" hks_status hks_shard_ks_inner_pipelined(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                                  const uint64_t *yall, const void *const *digit_ready,
                                                  const uint64_t *c1_loc, const uint64_t *evk_loc, uint32_t evk_digits,
                                                  uint64_t *acc_loc, uint64_t *ypsend, void *ws, void *stream) {
    if (!yall || !digit_ready) HKS_FAIL(HKS_EINVAL, "shard_ks_inner_pipelined: NULL yall / event table");
    return shard_inner(c, level, world, rank, yall, nullptr, c1_loc, evk_loc, evk_digits, acc_loc, ypsend, ws, stream,
                       digit_ready);
}

extern "C" hks_status hks_shard_ks_inner_peer(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                             const uint64_t *const *ysend_ranks, const uint64_t *c1_loc,
                                             const uint64_t *evk_loc, uint32_t evk_digits, uint64_t *acc_loc,
                                             uint64_t *ypsend, void *ws, void *stream) {
    if (!ysend_ranks) HKS_FAIL(HKS_EINVAL, "shard_ks_inner_peer: NULL rank table");
    return shard_inner(c, level, world, rank, nullptr, ysend_ranks, c1_loc, evk_loc, evk_digits, acc_loc, ypsend, ws,
                       stream);
}

extern "C" hks_status hks_shard_ks_moddown_out(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                              const uint64_t *ypall, const uint64_t *acc_loc, const uint64_t *c0_loc,
                                              uint64_t *out0_loc, uint64_t *out1_loc, void *ws, void *stream) {
    if (!ypall) HKS_FAIL(HKS_EINVAL, "shard_ks_moddown_out: NULL ypall");
    return shard_moddown(c, level, world, rank, ypall, nullptr, acc_loc, c0_loc, out0_loc, out1_loc, ws, stream);
}

extern "C" hks_status hks_shard_ks_moddown_out_peer(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                                   const uint64_t *const *ypsend_ranks, const uint64_t *acc_loc,
                                                   const uint64_t *c0_loc, uint64_t *out0_loc, uint64_t *out1_loc,
                                                   void *ws, void *stream) {
    if (!ypsend_ranks) HKS_FAIL(HKS_EINVAL, "shard_ks_moddown_out_peer: NULL rank table");
    return shard_moddown(c, level, world, rank, nullptr, ypsend_ranks, acc_loc, c0_loc, out0_loc, out1_loc, ws,
                         stream);
}

// ------------------------------------------------------------------------------------------------
// All-to-all coefficient-sharded KeySwitch (SURVEY.md §8(e) "coefficient-sharded BConv", §8(f) NEXT-3;
// include/hks.h).  Same limb ownership as above; the base conversions run on a coefficient chunk of EVERY
// limb instead of on every coefficient of the owned limbs, so each rank receives its chunk of the sources
// (all-to-all #1 / #3) and then the converted chunks of its owned targets (all-to-all #2 / #4).  Rank k's
// chunk = rows [k R / G, (k + 1) R / G) of the R x C limb layout (chunked layout: internal.h).
namespace {
struct A2A {
    u32 G, logG, clog, nc;     // world, log2 world, log2 rows per chunk, words per chunk of a limb
    u32 n_pad, nq_pad;         // max owned extended / active chain limbs over the ranks
};

hks_status make_a2a(const hks_ctx *c, const Plan &P, A2A &X) {
    X.G = P.world;
    X.logG = 0;
    while ((1u << X.logG) < X.G) X.logG++;
    if ((1u << X.logG) != X.G || X.logG > c->log_r) HKS_FAIL(HKS_EINVAL, "shard_a2a: world %u must be a power of two <= R", X.G);
    X.clog = c->log_r - X.logG;
    X.nc = c->n >> X.logG;
    X.n_pad = X.nq_pad = 0;
    for (u32 r = 0; r < P.world; r++) {
        const u32 nq = P.qlo_r[r] >= P.level + 1 ? 0 : std::min(P.qhi_r[r], P.level + 1) - P.qlo_r[r];
        X.nq_pad = std::max(X.nq_pad, nq);
        X.n_pad = std::max(X.n_pad, nq + (P.phi_r[r] - P.plo_r[r]));
    }
    return HKS_OK;
}

// local index of extended limb t (chain t <= level, or P_{t - level - 1}) in its owner's list (active chain
// limbs, then special limbs), and the owner
void ext_owner(const Plan &P, u32 level, u32 t, u32 &owner, u32 &u) {
    if (t <= level) {
        owner = P.q_owner(t);
        u = t - P.qlo_r[owner];
    } else {
        const u32 k = t - level - 1;
        owner = P.p_owner(k);
        const u32 nq = P.qlo_r[owner] >= level + 1 ? 0 : std::min(P.qhi_r[owner], level + 1) - P.qlo_r[owner];
        u = nq + (k - P.plo_r[owner]);
    }
}

// inverse NTT of L (in -> chunked out): row pass into scratch, column pass with the chunked store
hks_status intt_chunked(const hks_ctx *c, const LimbList &L, const u64 *in, u64 *scratch, u64 *out, u32 clog,
                        u64 cstride, const ulonglong2 *scale, u32 scale_mod, cudaStream_t s) {
    if (L.size() > HKS_MAXB) HKS_FAIL(HKS_EINVAL, "shard_a2a: batch larger than one launch");
    NttArgs a{};
    a.pc = c->d_pc;
    a.ninv = c->d_ninv;
    a.galois = 1;
    for (u32 i = 0; i < L.size(); i++) {
        a.map.sin[i] = L.sin[i];
        a.map.sout[i] = (u16)i;
        a.map.prime[i] = L.prime[i];
    }
    a.nlimbs = (u32)L.size();
    a.in = in;
    a.out = scratch;
    a.tw = c->d_tw_row_inv;
    hks_status st = launch_ntt_pass(c, NTT_INV, 0, EPI_LAZY, a, s);
    if (st != HKS_OK) return st;
    for (u32 i = 0; i < L.size(); i++) {
        a.map.sin[i] = (u16)i;
        a.map.sout[i] = L.sout[i];
    }
    a.in = scratch;
    a.out = out;
    a.tw = c->d_tw_col_inv;
    a.scale = scale;
    a.scale_mod = scale_mod ? scale_mod : 1;
    a.clog = clog;
    a.cstride = cstride;
    return launch_ntt_pass(c, NTT_INV, 1, EPI_SCALE_COUT, a, s);
}
}  // namespace

extern "C" hks_status hks_shard_a2a_query(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                          hks_shard_a2a_info *out) {
    if (!out) HKS_FAIL(HKS_EINVAL, "shard_a2a_query: NULL out");
    Plan P;
    A2A X;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = make_a2a(c, P, X)) != HKS_OK) return st;
    out->chunk_words = X.nc;
    out->n_pad = X.n_pad;
    out->nq_pad = X.nq_pad;
    out->beta = c->beta(level);
    return HKS_OK;
}

extern "C" size_t hks_shard_a2a_workspace_bytes(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank) {
    Plan P;
    A2A X;
    if (make_plan(c, level, world, rank, P) != HKS_OK || make_a2a(c, P, X) != HKS_OK) return 0;
    // ext [beta][n_own] | conv [2][nq_act] | scratch for the chunked inverse NTTs max(q_pad, 2 np_own)
    const size_t scratch = std::max<size_t>(P.q_pad, 2 * (size_t)P.np_own);
    return ((size_t)c->beta(level) * P.n_own + 2 * (size_t)P.nq_act + scratch) * c->n * sizeof(u64);
}

// #1 in: ysend [G][q_pad][Nc] = chunks of INTT(c1_loc) * N^-1 [qhat]^-1 (owned active chain limbs)
extern "C" hks_status hks_shard_a2a_modup_in(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                             const uint64_t *c1_loc, uint64_t *ysend, void *ws, void *stream) {
    Plan P;
    A2A X;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = make_a2a(c, P, X)) != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if (P.nq_act == 0) return HKS_OK;
    if (!c1_loc || !ysend || !ws) HKS_FAIL(HKS_EINVAL, "shard_a2a_modup_in: NULL buffer");
    DevGuard g(c->device);
    u64 *scratch = (u64 *)ws + ((size_t)c->beta(level) * P.n_own + 2 * (size_t)P.nq_act) * c->n;
    LimbList L;
    for (u32 li = 0; li < P.nq_act; li++) L.push(li, li, P.q_lo + li);
    return intt_chunked(c, L, c1_loc, scratch, ysend, X.clog, (u64)P.q_pad * X.nc,
                        c->d_mu_scale + c->mu_scale_off[level] + P.q_lo, P.nq_act, (cudaStream_t)stream);
}

// #1 out -> #2 in: yrecv [G][q_pad][Nc] (rank r's limbs at r) -> extsend [G][beta][n_pad][Nc]: for every digit
// j, Eq. 1 on this rank's coefficient chunk to every extended limb outside the digit, placed for its owner
extern "C" hks_status hks_shard_a2a_bconv(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                          const uint64_t *yrecv, uint64_t *extsend, void *stream) {
    Plan P;
    A2A X;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = make_a2a(c, P, X)) != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if (!yrecv || !extsend) HKS_FAIL(HKS_EINVAL, "shard_a2a_bconv: NULL buffer");
    const u32 beta = c->beta(level), ne = c->ne(level);
    if ((size_t)world * beta * X.n_pad > 0xffff) HKS_FAIL(HKS_EINVAL, "shard_a2a_bconv: too many slots");
    DevGuard g(c->device);
    std::vector<BconvGroup> groups;
    for (u32 j = 0; j < beta; j++) {
        const u32 lo = c->digit_lo(j), hi = c->digit_hi(level, j);
        u16 src[BC_MAXSRC];
        for (u32 i = lo; i < hi; i++) {
            const u32 r = P.q_owner(i);
            src[i - lo] = (u16)(r * P.q_pad + (i - P.qlo_r[r]));
        }
        std::vector<u16> ds, dp;
        for (u32 t = 0; t < ne; t++) {
            if (t >= lo && t < hi) continue;
            u32 d, u;
            ext_owner(P, level, t, d, u);
            ds.push_back((u16)(d * beta * X.n_pad + j * X.n_pad + u));
            dp.push_back((u16)c->ext_prime(level, t));
        }
        const size_t moff = c->mu_mat_off[(size_t)level * c->dnum + j];
        push_group(groups, hi - lo, src, c->d_mu_mat + moff, (u32)ds.size(), ds, dp, tab_at(c->d_mu_matf, 3 * moff),
                   c->d_mu_mats + moff, tab_at(c->d_mu_matb, 8 * moff),
                   c->d_mu_img + c->mu_img_off[(size_t)level * c->dnum + j]);
    }
    // the conversion kernels address limbs of Nc words: log N of a chunk
    std::vector<BconvGroup> gs(groups);
    size_t i = 0;
    while (i < gs.size()) {
        BconvArgs a{};
        a.in = yrecv;
        a.out = extsend;
        a.pc = c->d_pc;
        a.log_n = c->log_n - X.logG;
        a.lazy_out = 1;
        a.big = c->all_big ? 1 : 0;
        u32 ns = gs[i].nsrc, k = 0;
        while (i < gs.size() && k < BC_MAXG && gs[i].nsrc == ns) a.g[k++] = gs[i++];
        a.ngroups = k;
        if ((st = launch_bconv(a, BC_MAXDST, (cudaStream_t)stream)) != HKS_OK) return st;
    }
    return HKS_OK;
}

// #2 out -> #3 in: extrecv [G][beta][n_pad][Nc] (chunk r of the owned extended limbs) -> NTT, key inner product
// -> acc_loc; ypsend [G][2][p_pad][Nc] = chunks of INTT(acc_loc[P]) * N^-1 [phat]^-1
extern "C" hks_status hks_shard_a2a_inner(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                          const uint64_t *extrecv, const uint64_t *c1_loc, const uint64_t *evk_loc,
                                          uint32_t evk_digits, uint64_t *acc_loc, uint64_t *ypsend, void *ws,
                                          void *stream) {
    Plan P;
    A2A X;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = make_a2a(c, P, X)) != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if (!extrecv || !evk_loc || !acc_loc || !ypsend || !ws || (P.nq_act && !c1_loc))
        HKS_FAIL(HKS_EINVAL, "shard_a2a_inner: NULL buffer");
    const u32 beta = c->beta(level);
    if (beta > FK_MAXD) HKS_FAIL(HKS_EINVAL, "shard_a2a_inner: beta %u > %d", beta, FK_MAXD);
    if (evk_digits < beta || evk_digits > c->dnum)
        HKS_FAIL(HKS_EKEY, "shard_a2a_inner: key has %u digits; level %u needs %u (context dnum %u)", evk_digits, level,
                 beta, c->dnum);
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    u64 *ext = (u64 *)ws;
    u64 *scratch = ext + ((size_t)beta * P.n_own + 2 * (size_t)P.nq_act) * c->n;
    std::vector<u32> own_t;
    for (u32 li = 0; li < P.nq_act; li++) own_t.push_back(P.q_lo + li);
    for (u32 k = P.p_lo; k < P.p_hi; k++) own_t.push_back(level + 1 + k);
    // forward column pass of every converted (digit, owned target) limb, from the chunked receive buffer
    LimbList T;
    for (u32 j = 0; j < beta; j++) {
        const u32 lo = c->digit_lo(j), hi = c->digit_hi(level, j);
        for (u32 u = 0; u < own_t.size(); u++) {
            const u32 t = own_t[u];
            if (t >= lo && t < hi) continue;
            T.push(j * X.n_pad + u, j * P.n_own + u, c->ext_prime(level, t));
        }
    }
    for (size_t off = 0; off < T.size(); off += HKS_MAXB) {
        const u32 cnt = (u32)std::min<size_t>(HKS_MAXB, T.size() - off);
        NttArgs a{};
        a.pc = c->d_pc;
        a.ninv = c->d_ninv;
        a.galois = 1;
        for (u32 i = 0; i < cnt; i++) {
            a.map.sin[i] = T.sin[off + i];
            a.map.sout[i] = T.sout[off + i];
            a.map.prime[i] = T.prime[off + i];
        }
        a.nlimbs = cnt;
        a.in = extrecv;
        a.out = ext;
        a.tw = c->d_tw_col_fwd;
        a.clog = X.clog;
        a.cstride = (u64)beta * X.n_pad * X.nc;
        if ((st = launch_ntt_pass(c, NTT_FWD, 0, EPI_LAZY_CIN, a, s)) != HKS_OK) return st;
    }
    std::vector<KipItem> items(own_t.size());
    for (u32 u = 0; u < own_t.size(); u++) {
        const u32 t = own_t[u];
        KipItem &it = items[u];
        it.prime = (u16)c->ext_prime(level, t);
        it.kslot = (u16)(t <= level ? t - P.q_lo : (P.q_hi - P.q_lo) + (t - level - 1 - P.p_lo));
        it.aslot = (u16)u;
        for (u32 j = 0; j < beta; j++) {
            const bool own = t <= level && t >= c->digit_lo(j) && t < c->digit_hi(level, j);
            it.src[j] = own ? (u16)(FK_DIRECT | (t - P.q_lo)) : (u16)(j * P.n_own + u);
        }
    }
    if ((st = run_ntt_kip(c, items, beta, ext, c1_loc, evk_loc, acc_loc, P.nkey, P.n_own, s)) != HKS_OK) return st;
    if (P.np_own) {
        LimbList L;
        for (u32 p = 0; p < 2; p++)
            for (u32 kk = 0; kk < P.np_own; kk++) L.push(p * P.n_own + P.nq_act + kk, p * P.p_pad + kk, c->nq + P.p_lo + kk);
        if ((st = intt_chunked(c, L, acc_loc, scratch, ypsend, X.clog, (u64)2 * P.p_pad * X.nc, c->d_md_scale + P.p_lo,
                               P.np_own, s)) != HKS_OK)
            return st;
    }
    return HKS_OK;
}

// #3 out -> #4 in: yprecv [G][2][p_pad][Nc] -> convsend [G][2][nq_pad][Nc]: Eq. 1 P -> every active chain limb on
// this rank's chunk, placed for the chain limb's owner
extern "C" hks_status hks_shard_a2a_moddown_bconv(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                                  const uint64_t *yprecv, uint64_t *convsend, void *stream) {
    Plan P;
    A2A X;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = make_a2a(c, P, X)) != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if (!yprecv || !convsend) HKS_FAIL(HKS_EINVAL, "shard_a2a_moddown_bconv: NULL buffer");
    const u32 K = c->np;
    DevGuard g(c->device);
    std::vector<BconvGroup> groups;
    for (u32 p = 0; p < 2; p++) {
        u16 src[BC_MAXSRC];
        for (u32 k = 0; k < K; k++) {
            const u32 r = P.p_owner(k);
            src[k] = (u16)(r * 2 * P.p_pad + p * P.p_pad + (k - P.plo_r[r]));
        }
        std::vector<u16> ds(level + 1), dp(level + 1);
        for (u32 i = 0; i <= level; i++) {
            const u32 d = P.q_owner(i);
            ds[i] = (u16)(d * 2 * X.nq_pad + p * X.nq_pad + (i - P.qlo_r[d]));
            dp[i] = (u16)i;
        }
        push_group(groups, K, src, c->d_md_mat, c->nq, ds, dp, c->d_md_matf, c->d_md_mats, c->d_md_matb, c->d_md_img);
    }
    BconvArgs a{};
    a.in = yprecv;
    a.out = convsend;
    a.pc = c->d_pc;
    a.log_n = c->log_n - X.logG;
    a.lazy_out = 1;
    a.big = c->all_big ? 1 : 0;
    for (size_t k = 0; k < groups.size(); k++) a.g[k] = groups[k];
    a.ngroups = (u32)groups.size();
    return launch_bconv(a, BC_MAXDST, (cudaStream_t)stream);
}

// #4 out: convrecv [G][2][nq_pad][Nc] (chunk r of this rank's conv limbs) -> out_p = (acc_p - NTT(conv_p)) P^-1
// (+ c0 on p = 0) for the owned active chain limbs
extern "C" hks_status hks_shard_a2a_moddown_out(const hks_ctx *c, uint32_t level, uint32_t world, uint32_t rank,
                                                const uint64_t *convrecv, const uint64_t *acc_loc, const uint64_t *c0_loc,
                                                uint64_t *out0_loc, uint64_t *out1_loc, void *ws, void *stream) {
    Plan P;
    A2A X;
    hks_status st = make_plan(c, level, world, rank, P);
    if (st != HKS_OK || (st = make_a2a(c, P, X)) != HKS_OK || (st = dev_ctx(c)) != HKS_OK) return st;
    if (P.nq_act == 0) return HKS_OK;
    if (!convrecv || !acc_loc || !out0_loc || !out1_loc || !ws) HKS_FAIL(HKS_EINVAL, "shard_a2a_moddown_out: NULL buffer");
    DevGuard g(c->device);
    u64 *conv = (u64 *)ws + (size_t)c->beta(level) * P.n_own * c->n;
    LimbList M;
    std::vector<uint8_t> poly;
    ChunkIn cin{convrecv, X.clog, (u64)2 * X.nq_pad * X.nc, {}};
    for (u32 p = 0; p < 2; p++)
        for (u32 li = 0; li < P.nq_act; li++) {
            M.push(p * P.nq_act + li, li, P.q_lo + li, p * P.n_own + li, (p == 0 && c0_loc) ? li : 0xffff);
            poly.push_back((uint8_t)p);
            cin.slot.push_back((u16)(p * X.nq_pad + li));
        }
    std::vector<MdOut> mo = {MdOut{out0_loc, c0_loc, 1}, MdOut{out1_loc, nullptr, 1}};
    return run_ntt_moddown(c, M, poly, mo, conv, acc_loc, (cudaStream_t)stream, nullptr, &cin);
}
