// capi.cu -- the extern "C" entry points of include/hks.h and the key-switching orchestration.
//
// KeySwitch at level l (§2.1, 287-322 §3.6.3, 343-352 §3.6.5):
//   1. INTT(c1) with the Eq. 1 scale N^-1 [qhat_{j,i}]^-1 fused into the last pass   -> y (canonical)
//   2. BConv per digit j: y[digit j] -> every other extended limb                    (COEFF)
//   3. NTT of the beta(l+1+K) - (l+1) new limbs                                       (EVAL)
//   4. key inner product (own-digit limbs read straight from c1, EVAL)               -> acc0, acc1
//   5. ModDown of both: INTT(acc_P) with N^-1 [phat_k]^-1 fused, BConv P -> Q_l, NTT with the fused
//      epilogue out = (acc - NTT(conv)) P^-1 (+ c0)
// All launches go to the caller's stream; the workspace is caller-owned.
#include <string.h>

#include <algorithm>

#include "internal.h"

namespace {

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

hks_status check_ctx(const hks_ctx *c) {
    if (!c) HKS_FAIL(HKS_EINVAL, "NULL context");
    if (c->device < 0) HKS_FAIL(HKS_EDEVICE, "host-only context cannot run device operations");
    return HKS_OK;
}

bool overlap(const void *a, size_t na, const void *b, size_t nb) {
    if (!a || !b || !na || !nb) return false;
    const char *x = (const char *)a, *y = (const char *)b;
    return x < y + nb && y < x + na;
}

size_t limb_bytes(const hks_ctx *c) { return (size_t)c->n * sizeof(u64); }

// Launch BConv groups, batching up to BC_MAXG groups with equal nsrc per launch.
hks_status run_bconv_groups(const hks_ctx *c, std::vector<BconvGroup> &groups, const u64 *in, u64 *out,
                            cudaStream_t s) {
    size_t i = 0;
    while (i < groups.size()) {
        BconvArgs a{};
        a.in = in;
        a.out = out;
        a.pc = c->d_pc;
        a.log_n = c->log_n;
        a.lazy_out = 1;   // internal conversions feed the forward NTT, which takes [0, 8p + 2^32)
        a.big = c->all_big ? 1 : 0;
        u32 ns = groups[i].nsrc, k = 0;
        while (i < groups.size() && k < BC_MAXG && groups[i].nsrc == ns) a.g[k++] = groups[i++];
        a.ngroups = k;
        hks_status st = launch_bconv(a, BC_MAXDST, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}

// groups converting src slots -> dst slots with a row-major matrix [nsrc][stride]; targets chunked by 64
void add_groups(std::vector<BconvGroup> &out, u32 nsrc, const u16 *src_slot, const uint2 *mat, u32 stride,
                const std::vector<u16> &dst_slot, const std::vector<u16> &dst_prime, const double *matf = nullptr,
                const u32 *mats = nullptr, const u64 *matb = nullptr, const u64 *mimg = nullptr) {
    for (size_t u0 = 0; u0 < dst_slot.size(); u0 += BC_MAXDST) {
        BconvGroup g{};
        g.nsrc = nsrc;
        g.ndst = (u32)std::min<size_t>(BC_MAXDST, dst_slot.size() - u0);
        g.mat_stride = stride;
        g.mat = mat + u0;
        g.matf = matf ? matf + 3 * u0 : nullptr;   // NULL unless HKS_EXPERIMENTAL uploaded the table
        g.mats = mats ? mats + u0 : nullptr;
        g.matb = matb ? matb + 8 * u0 : nullptr;
        g.mimg = mimg ? mimg + (size_t)bconv_img_words(nsrc) * u0 : nullptr;
        for (u32 i = 0; i < nsrc; i++) g.src_slot[i] = src_slot[i];
        for (u32 u = 0; u < g.ndst; u++) {
            g.dst_slot[u] = dst_slot[u0 + u];
            g.dst_prime[u] = dst_prime[u0 + u];
        }
        out.push_back(g);
    }
}

// ModUp: d [l+1][N] EVAL -> ext slots (j * ne + t) for t outside digit j.  coef: [l+1][N] scratch.
// rows_pass = false stops after the column pass of the forward NTT (the KeySwitch fuses the row
// pass with the key inner product).
// d_b != NULL (HMult): the input is the tensor term d * d_b, computed inside the first INTT pass and
// also stored (EVAL) to d_side for the key product's own-digit limbs.
hks_status modup_core(const hks_ctx *c, const u64 *d, u32 level, u64 *ext, u64 *coef, cudaStream_t s,
                      bool rows_pass = true, const u64 *d_b = nullptr, u64 *d_side = nullptr) {
    const u32 ne = c->ne(level), beta = c->beta(level);
    LimbList L;
    for (u32 i = 0; i <= level; i++) L.push(i, i, i);
    hks_status st = run_ntt(c, NTT_INV, L, d, coef, c->d_mu_scale + c->mu_scale_off[level], level + 1, s, d_b, d_side);
    if (st != HKS_OK) return st;
    std::vector<BconvGroup> groups;
    LimbList T;
    for (u32 j = 0; j < beta; j++) {
        u32 lo = c->digit_lo(j), hi = c->digit_hi(level, j);
        u16 src[BC_MAXSRC];
        for (u32 i = lo; i < hi; i++) src[i - lo] = (u16)i;
        std::vector<u16> ds, dp;
        for (u32 t = 0; t < ne; t++) {
            if (t >= lo && t < hi) continue;
            ds.push_back((u16)(j * ne + t));
            dp.push_back((u16)c->ext_prime(level, t));
            T.push(j * ne + t, j * ne + t, c->ext_prime(level, t));
        }
        const size_t off = c->mu_mat_off[(size_t)level * c->dnum + j];
        add_groups(groups, hi - lo, src, c->d_mu_mat + off, (u32)ds.size(), ds, dp, tab_at(c->d_mu_matf, 3 * off),
                   c->d_mu_mats + off, tab_at(c->d_mu_matb, 8 * off), c->d_mu_img + c->mu_img_off[(size_t)level * c->dnum + j]);
    }
    st = run_bconv_groups(c, groups, coef, ext, s);
    if (st != HKS_OK) return st;
    if (!rows_pass) return run_ntt_fwd_cols(c, T, ext, ext, s);
    return run_ntt(c, NTT_FWD, T, ext, ext, nullptr, 0, s);
}

// Fused row pass + key inner product for the KeySwitch (own-digit limbs read from c1, EVAL).
// y != NULL: P-limb tiles also run ModDown's first inverse-NTT pass and write it to y [2][K][N]
// (needs beta >= 2: two thread groups for the two accumulators).
hks_status ntt_kip_core(const hks_ctx *c, const u64 *ext, const u64 *c1, const u64 *evk, u32 level, u64 *acc,
                        cudaStream_t s, u64 *y = nullptr) {
    const u32 ne = c->ne(level), beta = c->beta(level);
    std::vector<KipItem> items(ne);
    for (u32 t = 0; t < ne; t++) {
        KipItem &it = items[t];
        it.prime = it.kslot = (u16)c->ext_prime(level, t);
        it.aslot = (u16)t;
        if (y && t > level) it.yslot = (u16)(t - level - 1);
        for (u32 j = 0; j < beta; j++) {
            const bool own = t <= level && t >= c->digit_lo(j) && t < c->digit_hi(level, j);
            it.src[j] = own ? (u16)(FK_DIRECT | t) : (u16)(j * ne + t);
        }
    }
    return run_ntt_kip(c, items, beta, ext, c1, evk, acc, c->nq + c->np, ne, s, y, c->np);
}

// ModDown of npoly accumulators (acc poly p at slots p * ne + t) into outs[p], + adds[p] read through
// the automorphism gal[p].  ws: y [npoly][K][N] then conv [npoly][l+1][N].  y_rows_done: the inverse
// row pass of the P limbs already ran inside k_ntt_kip (y holds it).
// prepared: the accumulators come from a key prepared by hks_evk_prepare (Q limbs times P^-1): the conversion
// uses the P^-1-folded matrix and the epilogue skips its P^-1 product (bit-identical outputs)
hks_status moddown_core(const hks_ctx *c, const u64 *acc, u32 npoly, u32 level, u64 *const *outs,
                        const u64 *const *adds, const u64 *gal, u64 *ws, cudaStream_t s, bool y_rows_done = false,
                        const u64 *const *tensor = nullptr, bool prepared = false) {
    const u32 ne = c->ne(level), K = c->np;
    u64 *y = ws, *conv = ws + (size_t)npoly * K * c->n;
    hks_status st = HKS_OK;
    // inverse NTT of the P limbs with N^-1 [phat_k]^-1 (one launch pair per HKS_MAXB limbs)
    for (u32 p0 = 0; p0 < npoly && st == HKS_OK;) {
        const u32 np = std::min<u32>(npoly - p0, HKS_MAXB / K);
        LimbList L;
        for (u32 p = p0; p < p0 + np; p++)
            for (u32 k = 0; k < K; k++)
                L.push(y_rows_done ? p * K + k : p * ne + level + 1 + k, p * K + k, c->nq + k);
        st = y_rows_done ? run_ntt_inv_cols(c, L, y, y, c->d_md_scale, K, s)
                         : run_ntt(c, NTT_INV, L, acc, y, c->d_md_scale, K, s);
        p0 += np;
    }
    if (st != HKS_OK) return st;
    std::vector<BconvGroup> groups;
    std::vector<u16> dp(level + 1);
    for (u32 i = 0; i <= level; i++) dp[i] = (u16)i;
    for (u32 p = 0; p < npoly; p++) {
        u16 src[BC_MAXSRC];
        for (u32 k = 0; k < K; k++) src[k] = (u16)(p * K + k);
        std::vector<u16> ds(level + 1);
        for (u32 i = 0; i <= level; i++) ds[i] = (u16)(p * (level + 1) + i);
        if (prepared)
            add_groups(groups, K, src, c->d_mdp_mat, c->nq, ds, dp, c->d_mdp_matf, c->d_mdp_mats, c->d_mdp_matb,
                       c->d_mdp_img);
        else
            add_groups(groups, K, src, c->d_md_mat, c->nq, ds, dp, c->d_md_matf, c->d_md_mats, c->d_md_matb, c->d_md_img);
    }
    st = run_bconv_groups(c, groups, y, conv, s);
    if (st != HKS_OK) return st;
    LimbList M;
    std::vector<uint8_t> poly;
    std::vector<MdOut> mo(npoly);
    for (u32 p = 0; p < npoly; p++) mo[p] = MdOut{outs[p], adds ? adds[p] : nullptr, gal ? gal[p] : 1};
    // limb-major when one launch can take every polynomial (NTT_MAXO): the polynomials' limbs of one prime are
    // adjacent in the launch, so the CTAs that read a prime's per-row twiddle table run together and share it
    // in L2
    const bool lm = npoly <= NTT_MAXO;
    for (u32 a = 0; a < (lm ? level + 1 : npoly); a++)
        for (u32 b = 0; b < (lm ? npoly : level + 1); b++) {
            const u32 i = lm ? a : b, p = lm ? b : a;
            M.push(p * (level + 1) + i, i, i, p * ne + i, mo[p].add ? i : 0xffff);
            poly.push_back((uint8_t)p);
        }
    return run_ntt_moddown(c, M, poly, mo, conv, acc, s, tensor, nullptr, prepared);
}

hks_status kip_core(const hks_ctx *c, const u64 *ext, const u64 *c1, const u64 *evk, u32 level, u64 galois,
                    u64 *acc, cudaStream_t s) {
    KipArgs a{};
    a.ext = ext;
    a.c1 = c1;
    a.evk = evk;
    a.acc = acc;
    a.pc = c->d_pc;
    a.galois = galois;
    a.log_n = c->log_n;
    a.level = level;
    a.nq = c->nq;
    a.np = c->np;
    a.ne = c->ne(level);
    a.nk = c->nq + c->np;
    a.beta = c->beta(level);
    a.alpha = c->alpha;
    return launch_kip(a, s);
}

// rotations whose ModDowns are batched together: 2 RB polynomials must fit the 16-entry output
// table of one ModDown epilogue launch and the K-limb INTT batches (HKS_MAXB limbs).
// branches of hks_rotate_hoisted: the rotations after the shared ModUp split over the caller's stream and
// the context's side streams (one branch for a single rotation or a host-only context)
size_t rot_branches(const hks_ctx *c, u32 nrot) {
    return (nrot > 1 && c->side[0]) ? std::min<size_t>(1 + hks_ctx::NSIDE, nrot) : 1;
}

size_t rot_batch(const hks_ctx *c, u32 level) {
    (void)level;
    return std::max<size_t>(1, std::min<size_t>(NTT_MAXO / 2, HKS_MAXB / (2 * c->np)));
}

// the key's digit count (include/hks.h "Keys"): a call at `level` reads digits 0..beta(level)-1
// HKS_EVK_PREPARED in evk_digits marks a key from hks_evk_prepare
static bool evk_prepared(u32 evk_digits) { return (evk_digits & HKS_EVK_PREPARED) != 0; }
hks_status check_evk(const hks_ctx *c, u32 evk_digits, u32 level, const char *where) {
    evk_digits &= ~HKS_EVK_PREPARED;
    if (evk_digits < c->beta(level) || evk_digits > c->dnum)
        HKS_FAIL(HKS_EKEY, "%s: key has %u digits; level %u needs %u (context dnum %u)", where, evk_digits, level,
                 c->beta(level), c->dnum);
    return HKS_OK;
}
size_t evk_bytes(const hks_ctx *c, u32 evk_digits) {
    return (size_t)(evk_digits & ~HKS_EVK_PREPARED) * 2 * (c->nq + c->np) * limb_bytes(c);
}

// Fork / join of the context's side streams around the independent branches of one call.  join() -- also
// run by the destructor when a branch returns an error -- records every forked side stream's join event and
// makes the caller's stream wait on it, so work already enqueued on a side stream stays ordered before
// whatever the caller enqueues next, and a stream capture ends joined.
struct SideFork {
    const hks_ctx *c;
    cudaStream_t s;
    int nb = 1;
    bool joined = true;
    std::unique_lock<std::recursive_mutex> lk;
    SideFork(const hks_ctx *c_, cudaStream_t s_) : c(c_), s(s_), lk(c_->side_mu, std::defer_lock) {}
    cudaStream_t stream(int b) const { return b == 0 ? s : c->side[b - 1]; }
    hks_status fork(int n, const char *where) {
        if (n <= 1) return HKS_OK;
        lk.lock();
        if (cudaEventRecord(c->ev_fork, s) != cudaSuccess) HKS_FAIL(HKS_ECUDA, "%s: fork event record", where);
        joined = false;
        for (nb = 1; nb < n; nb++)
            if (cudaStreamWaitEvent(c->side[nb - 1], c->ev_fork, 0) != cudaSuccess) HKS_FAIL(HKS_ECUDA, "%s: fork wait", where);
        return HKS_OK;
    }
    bool join_quiet() {
        if (joined) return true;
        joined = true;
        bool ok = true;
        for (int b = 1; b < nb; b++)
            ok &= cudaEventRecord(c->ev_join[b - 1], c->side[b - 1]) == cudaSuccess &&
                  cudaStreamWaitEvent(s, c->ev_join[b - 1], 0) == cudaSuccess;
        return ok;
    }
    hks_status join(const char *where) {
        if (!join_quiet()) HKS_FAIL(HKS_ECUDA, "%s: join", where);
        return HKS_OK;
    }
    ~SideFork() { (void)join_quiet(); }
};

hks_status check_galois(const hks_ctx *c, u64 g) {
    if ((g & 1) == 0 || g >= 2 * (u64)c->n) HKS_FAIL(HKS_EGALOIS, "galois element %llu must be odd and < 2N", (unsigned long long)g);
    return HKS_OK;
}

}  // namespace

extern "C" size_t hks_workspace_bytes(const hks_ctx *c, hks_op op, uint32_t level, uint32_t count) {
    if (!c || level > c->L()) return 0;
    const size_t lb = limb_bytes(c), l1 = level + 1, ne = c->ne(level), K = c->np, beta = c->beta(level);
    switch (op) {
        case HKS_OP_MODUP: return l1 * lb;
        case HKS_OP_MODDOWN: return (K + l1) * lb;
        case HKS_OP_KEYSWITCH: return (l1 + beta * ne + 2 * ne + 2 * K + 2 * l1) * lb;
        case HKS_OP_ROTATE_HOISTED: {
            // count = 0: the worst case over every nrot (all branches, full rotation batches)
            const size_t nr = count ? count : (size_t)(1 + hks_ctx::NSIDE) * rot_batch(c, level);
            const size_t nb = rot_branches(c, (u32)nr);
            const size_t rb = std::min<size_t>((nr + nb - 1) / nb, rot_batch(c, level));
            return (l1 + beta * ne + nb * rb * (2 * ne + 2 * K + 2 * l1)) * lb;
        }
        case HKS_OP_HMULT: return (l1 + beta * ne + 2 * ne + 2 * K + 2 * l1 + l1) * lb;
        case HKS_OP_RESCALE: {
            if (level == 0) return 0;
            const size_t np_ = count ? count : 1;
            return (np_ + np_ * level) * lb;
        }
    }
    return 0;
}

extern "C" hks_status hks_ntt_fwd(const hks_ctx *c, uint64_t *x, const uint32_t *prime_idx, uint32_t nlimbs,
                                  void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!x || !prime_idx || nlimbs == 0) HKS_FAIL(HKS_EINVAL, "ntt_fwd: NULL buffer / empty batch");
    if (nlimbs > 0xffff) HKS_FAIL(HKS_EINVAL, "ntt_fwd: batch too large");
    LimbList L;
    for (u32 b = 0; b < nlimbs; b++) {
        if (prime_idx[b] >= c->primes.size()) HKS_FAIL(HKS_EINVAL, "ntt_fwd: prime index %u out of range", prime_idx[b]);
        L.push(b, b, prime_idx[b]);
    }
    DevGuard g(c->device);
    return run_ntt(c, NTT_FWD, L, x, x, nullptr, 0, (cudaStream_t)stream);
}

extern "C" hks_status hks_ntt_inv(const hks_ctx *c, uint64_t *x, const uint32_t *prime_idx, uint32_t nlimbs,
                                  void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!x || !prime_idx || nlimbs == 0) HKS_FAIL(HKS_EINVAL, "ntt_inv: NULL buffer / empty batch");
    if (nlimbs > 0xffff) HKS_FAIL(HKS_EINVAL, "ntt_inv: batch too large");
    LimbList L;
    for (u32 b = 0; b < nlimbs; b++) {
        if (prime_idx[b] >= c->primes.size()) HKS_FAIL(HKS_EINVAL, "ntt_inv: prime index %u out of range", prime_idx[b]);
        L.push(b, b, prime_idx[b]);
    }
    DevGuard g(c->device);
    return run_ntt(c, NTT_INV, L, x, x, nullptr, 0, (cudaStream_t)stream);
}

namespace {
// hks_bconv workspace (words): y [nsrc][N] | w, wp [2 * 16] | mat uint2 [nsrc][ndst] | img [ndst][img(nsrc)],
// every region 128-byte aligned
struct BconvWs {
    size_t y, w, mat, img, total;
    BconvWs(const hks_ctx *c, u32 nsrc, u32 ndst) {
        auto up = [](size_t x) { return (x + 15) & ~(size_t)15; };
        y = 0;
        w = up((size_t)nsrc * c->n);
        mat = w + up(2 * BC_MAXSRC);
        img = mat + up((size_t)nsrc * ndst);
        total = img + up((size_t)ndst * bconv_img_words(nsrc));
    }
};
}  // namespace

extern "C" size_t hks_bconv_workspace_bytes(const hks_ctx *c, uint32_t nsrc, uint32_t ndst) {
    if (!c || nsrc < 1 || nsrc > BC_MAXSRC || ndst < 1 || ndst > 2 * BC_MAXDST) return 0;
    return BconvWs(c, nsrc, ndst).total * sizeof(u64);
}

extern "C" hks_status hks_bconv(const hks_ctx *c, const uint64_t *x, const uint32_t *src_idx, uint32_t nsrc,
                                const uint32_t *dst_idx, uint32_t ndst, uint64_t *out, void *ws, void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!x || !out || !src_idx || !dst_idx || !ws) HKS_FAIL(HKS_EINVAL, "bconv: NULL argument");
    if (nsrc < 1 || nsrc > BC_MAXSRC || ndst < 1 || ndst > 2 * BC_MAXDST)
        HKS_FAIL(HKS_EINVAL, "bconv: nsrc must be in [1,%d], ndst in [1,%d]", BC_MAXSRC, 2 * BC_MAXDST);
    const size_t lb = limb_bytes(c);
    const BconvWs L(c, nsrc, ndst);
    if (overlap(x, nsrc * lb, out, ndst * lb) || overlap(ws, L.total * 8, out, ndst * lb) ||
        overlap(ws, L.total * 8, x, nsrc * lb))
        HKS_FAIL(HKS_EINVAL, "bconv: buffers overlap");
    const u32 nm = (u32)c->primes.size();
    u64 sp[BC_MAXSRC], dp[2 * BC_MAXDST];
    for (u32 i = 0; i < nsrc; i++) {
        if (src_idx[i] >= nm) HKS_FAIL(HKS_EINVAL, "bconv: src prime index out of range");
        for (u32 k = 0; k < i; k++)
            if (src_idx[k] == src_idx[i]) HKS_FAIL(HKS_EINVAL, "bconv: repeated source prime");
        sp[i] = c->primes[src_idx[i]];
    }
    for (u32 u = 0; u < ndst; u++) {
        if (dst_idx[u] >= nm) HKS_FAIL(HKS_EINVAL, "bconv: dst prime index out of range");
        for (u32 i = 0; i < nsrc; i++)
            if (src_idx[i] == dst_idx[u]) HKS_FAIL(HKS_EINVAL, "bconv: source and target bases overlap");
        dp[u] = c->primes[dst_idx[u]];
    }
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    u64 *w64 = (u64 *)ws;
    u64 *y = w64 + L.y, *w = w64 + L.w, *img = w64 + L.img;
    uint2 *mat = reinterpret_cast<uint2 *>(w64 + L.mat);
    // constants (device), y_i = [x_i qhat_i^-1]_{q_i} (canonical, reading 16), then the conversion kernel the
    // hot path uses for this shape (tcgen05 for large rings with primes > 2^49, else the integer pipe)
    if ((st = launch_bconv_prep(sp, nsrc, dp, ndst, w, mat, img, s)) != HKS_OK) return st;
    if ((st = launch_limb_scale(x, y, nsrc, w, sp, c->log_n, s)) != HKS_OK) return st;
    for (u32 u0 = 0; u0 < ndst; u0 += BC_MAXDST) {
        BconvArgs a{};
        a.in = y;
        a.out = out;
        a.pc = c->d_pc;
        a.log_n = c->log_n;
        a.lazy_out = 0;
        a.big = c->all_big ? 1 : 0;
        a.fresh_tables = 1;
        a.ngroups = 1;
        BconvGroup &G = a.g[0];
        G.nsrc = nsrc;
        G.ndst = std::min<u32>(BC_MAXDST, ndst - u0);
        G.mat_stride = ndst;
        G.mat = mat + u0;
        G.mimg = img + (size_t)bconv_img_words(nsrc) * u0;
        for (u32 i = 0; i < nsrc; i++) {
            G.src_slot[i] = (u16)i;
            G.src_prime[i] = (u16)src_idx[i];
        }
        for (u32 u = 0; u < G.ndst; u++) {
            G.dst_slot[u] = (u16)(u0 + u);
            G.dst_prime[u] = (u16)dst_idx[u0 + u];
        }
        if ((st = launch_bconv(a, BC_MAXDST, s)) != HKS_OK) return st;
    }
    return HKS_OK;
}

extern "C" hks_status hks_modup(const hks_ctx *c, const uint64_t *d, uint32_t level, uint64_t *ext, void *ws,
                                void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!d || !ext || !ws) HKS_FAIL(HKS_EINVAL, "modup: NULL argument");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "modup: level %u > L", level);
    const size_t lb = limb_bytes(c), ne = c->ne(level), beta = c->beta(level);
    if (overlap(d, (level + 1) * lb, ext, beta * ne * lb) || overlap(ws, (level + 1) * lb, ext, beta * ne * lb) ||
        overlap(ws, (level + 1) * lb, d, (level + 1) * lb))
        HKS_FAIL(HKS_EINVAL, "modup: buffers overlap");
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    st = modup_core(c, d, level, ext, (u64 *)ws, s);
    if (st != HKS_OK) return st;
    for (u32 j = 0; j < beta; j++) {
        u32 lo = c->digit_lo(j), hi = c->digit_hi(level, j);
        HKS_CUDA(cudaMemcpyAsync(ext + ((size_t)j * ne + lo) * c->n, d + (size_t)lo * c->n, (hi - lo) * lb,
                                 cudaMemcpyDeviceToDevice, s));
    }
    return HKS_OK;
}

extern "C" hks_status hks_ksk_inner_product(const hks_ctx *c, const uint64_t *ext, const uint64_t *evk,
                                            uint32_t evk_digits, uint32_t level, uint64_t galois, uint64_t *acc,
                                            void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!ext || !evk || !acc) HKS_FAIL(HKS_EINVAL, "ksk_inner_product: NULL argument");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "ksk_inner_product: level %u > L", level);
    if (galois != 1 && (st = check_galois(c, galois)) != HKS_OK) return st;
    if ((st = check_evk(c, evk_digits, level, "ksk_inner_product")) != HKS_OK) return st;
    if (evk_prepared(evk_digits))   // hks_moddown would apply P^-1 a second time
        HKS_FAIL(HKS_EINVAL, "ksk_inner_product: a prepared key (hks_evk_prepare) is for the fused calls only");
    const size_t lb = limb_bytes(c), ne = c->ne(level);
    if (overlap(ext, c->beta(level) * ne * lb, acc, 2 * ne * lb) || overlap(evk, evk_bytes(c, evk_digits), acc, 2 * ne * lb))
        HKS_FAIL(HKS_EINVAL, "ksk_inner_product: acc overlaps an input");
    DevGuard g(c->device);
    return kip_core(c, ext, nullptr, evk, level, galois, acc, (cudaStream_t)stream);
}

extern "C" hks_status hks_moddown(const hks_ctx *c, const uint64_t *acc, uint32_t level, uint64_t *out, void *ws,
                                  void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!acc || !out || !ws) HKS_FAIL(HKS_EINVAL, "moddown: NULL argument");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "moddown: level %u > L", level);
    const size_t lb = limb_bytes(c), ne = c->ne(level), wsb = (c->np + level + 1) * lb;
    if (overlap(acc, ne * lb, out, (level + 1) * lb) || overlap(ws, wsb, out, (level + 1) * lb) ||
        overlap(ws, wsb, acc, ne * lb))
        HKS_FAIL(HKS_EINVAL, "moddown: buffers overlap");
    DevGuard g(c->device);
    u64 *outs[1] = {out};
    return moddown_core(c, acc, 1, level, outs, nullptr, nullptr, (u64 *)ws, (cudaStream_t)stream);
}

static hks_status keyswitch_impl(const hks_ctx *c, const uint64_t *c0, const uint64_t *c1, const uint64_t *add1,
                                  uint32_t level, const uint64_t *evk, uint32_t evk_digits, uint64_t *out0,
                                  uint64_t *out1, void *ws, void *stream, const uint64_t *const *tensor = nullptr);

extern "C" hks_status hks_keyswitch(const hks_ctx *c, const uint64_t *c0, const uint64_t *c1, uint32_t level,
                                    const uint64_t *evk, uint32_t evk_digits, uint64_t *out0, uint64_t *out1, void *ws,
                                    void *stream) {
    return keyswitch_impl(c, c0, c1, nullptr, level, evk, evk_digits, out0, out1, ws, stream);
}

extern "C" hks_status hks_relinearize(const hks_ctx *c, const uint64_t *d0, const uint64_t *d1, const uint64_t *d2,
                                      uint32_t level, const uint64_t *evk, uint32_t evk_digits, uint64_t *out0,
                                      uint64_t *out1, void *ws, void *stream) {
    if (!d1) HKS_FAIL(HKS_EINVAL, "relinearize: NULL d1");
    if (c && level <= c->L() && (overlap(d1, (level + 1) * limb_bytes(c), out0, (level + 1) * limb_bytes(c)) ||
                                 overlap(d1, (level + 1) * limb_bytes(c), out1, (level + 1) * limb_bytes(c))))
        HKS_FAIL(HKS_EINVAL, "relinearize: d1 overlaps an output");
    return keyswitch_impl(c, d0, d2, d1, level, evk, evk_digits, out0, out1, ws, stream);
}

static hks_status keyswitch_impl(const hks_ctx *c, const uint64_t *c0, const uint64_t *c1, const uint64_t *add1,
                                  uint32_t level, const uint64_t *evk, uint32_t evk_digits, uint64_t *out0,
                                  uint64_t *out1, void *ws, void *stream, const uint64_t *const *tensor) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!c1 || !evk || !out0 || !out1 || !ws) HKS_FAIL(HKS_EINVAL, "keyswitch: NULL argument");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "keyswitch: level %u > L", level);
    if ((st = check_evk(c, evk_digits, level, "keyswitch")) != HKS_OK) return st;
    const size_t lb = limb_bytes(c), l1 = level + 1, ne = c->ne(level), beta = c->beta(level);
    const size_t wsb = hks_workspace_bytes(c, tensor ? HKS_OP_HMULT : HKS_OP_KEYSWITCH, level, 0);
    const void *ins[6] = {c0, c1, evk, tensor ? tensor[1] : nullptr, tensor ? tensor[2] : nullptr,
                          tensor ? tensor[3] : nullptr};
    size_t insz[6] = {l1 * lb, l1 * lb, evk_bytes(c, evk_digits), l1 * lb, l1 * lb, l1 * lb};
    void *outs_[3] = {out0, out1, ws};
    size_t outsz[3] = {l1 * lb, l1 * lb, wsb};
    for (int i = 0; i < 6; i++)
        for (int o = 0; o < 3; o++)
            if (overlap(ins[i], insz[i], outs_[o], outsz[o])) HKS_FAIL(HKS_EINVAL, "keyswitch: output overlaps an input");
    if (overlap(out0, l1 * lb, out1, l1 * lb) || overlap(out0, l1 * lb, ws, wsb) || overlap(out1, l1 * lb, ws, wsb))
        HKS_FAIL(HKS_EINVAL, "keyswitch: outputs overlap");
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    u64 *coef = (u64 *)ws;
    u64 *ext = coef + l1 * c->n;
    u64 *acc = ext + beta * ne * c->n;
    u64 *md = acc + 2 * ne * c->n;
    // HMult: d2 = a1 * b1 is formed inside the first INTT pass and kept (EVAL) after the ModDown
    // workspace for the key product's own-digit limbs
    u64 *d2 = tensor ? md + (2 * c->np + 2 * l1) * c->n : nullptr;
    const u64 *kin = tensor ? d2 : c1;
    const u64 *tb = tensor ? tensor[3] : nullptr;
    const bool fused = beta <= FK_MAXD;
    const bool ymode = fused && 2 * c->np <= HKS_MAXB;   // beta = 1: the launch gets a second thread group
    if (fused) {
        // INTT + BConv + NTT column pass, then the fused NTT row pass + key inner product (+ for the P
        // limbs, ModDown's inverse row pass straight into the ModDown workspace)
        if ((st = modup_core(c, c1, level, ext, coef, s, false, tb, d2)) != HKS_OK) return st;
        if ((st = ntt_kip_core(c, ext, kin, evk, level, acc, s, ymode ? md : nullptr)) != HKS_OK) return st;
    } else {
        if ((st = modup_core(c, c1, level, ext, coef, s, true, tb, d2)) != HKS_OK) return st;
        if ((st = kip_core(c, ext, kin, evk, level, 1, acc, s)) != HKS_OK) return st;
    }
    u64 *outs[2] = {out0, out1};
    const u64 *adds[2] = {c0, add1};
    const bool prep = evk_prepared(evk_digits);
    if (tensor) return moddown_core(c, acc, 2, level, outs, nullptr, nullptr, md, s, ymode, tensor, prep);
    return moddown_core(c, acc, 2, level, outs, adds, nullptr, md, s, ymode, nullptr, prep);
}

extern "C" hks_status hks_hmult(const hks_ctx *c, const uint64_t *a0, const uint64_t *a1, const uint64_t *b0,
                                const uint64_t *b1, uint32_t level, const uint64_t *evk, uint32_t evk_digits,
                                uint64_t *out0, uint64_t *out1, void *ws, void *stream) {
    if (!a0 || !a1 || !b0 || !b1) HKS_FAIL(HKS_EINVAL, "hmult: NULL ciphertext half");
    const uint64_t *tensor[4] = {a0, a1, b0, b1};
    // the KeySwitch input is d2 = a1 * b1 (first factor a1 passed as c1); a0 and c0 = NULL
    return keyswitch_impl(c, a0, a1, nullptr, level, evk, evk_digits, out0, out1, ws, stream, tensor);
}

extern "C" hks_status hks_rescale(const hks_ctx *c, const uint64_t *x, uint32_t npoly, uint32_t level, uint64_t *out,
                                  void *ws, void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!x || !out || !ws || npoly == 0) HKS_FAIL(HKS_EINVAL, "rescale: NULL argument / no polynomial");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "rescale: level %u > L", level);
    if (level == 0) HKS_FAIL(HKS_EINVAL, "rescale: level 0 has no limb to drop");
    if (npoly > 0xffff / (level + 1)) HKS_FAIL(HKS_EINVAL, "rescale: too many polynomials");
    const size_t lb = limb_bytes(c), wsb = hks_workspace_bytes(c, HKS_OP_RESCALE, level, npoly);
    const size_t xb = (size_t)npoly * (level + 1) * lb, ob = (size_t)npoly * level * lb;
    if (overlap(x, xb, out, ob) || overlap(ws, wsb, out, ob) || overlap(ws, wsb, x, xb))
        HKS_FAIL(HKS_EINVAL, "rescale: buffers overlap");
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    u64 *coef = (u64 *)ws, *buf = coef + (size_t)npoly * c->n;
    // INTT of every top limb (canonical COEFF), then the fused SwitchModulo / NTT / epilogue passes
    LimbList L;
    for (u32 p = 0; p < npoly; p++) L.push(p * (level + 1) + level, p, level);
    if ((st = run_ntt(c, NTT_INV, L, x, coef, nullptr, 0, s)) != HKS_OK) return st;
    std::vector<u64 *> outs(npoly);
    for (u32 p = 0; p < npoly; p++) outs[p] = out + (size_t)p * level * c->n;
    return run_rescale(c, npoly, level, x, coef, buf, outs.data(), s);
}

extern "C" hks_status hks_evk_prepare(const hks_ctx *c, const uint64_t *evk_in, uint32_t evk_digits, uint64_t *evk_out,
                                      void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!evk_in || !evk_out) HKS_FAIL(HKS_EINVAL, "evk_prepare: NULL key");
    if (evk_digits & HKS_EVK_PREPARED) HKS_FAIL(HKS_EINVAL, "evk_prepare: the key is already prepared");
    if (evk_digits == 0 || evk_digits > c->dnum)
        HKS_FAIL(HKS_EKEY, "evk_prepare: key has %u digits (context dnum %u)", evk_digits, c->dnum);
    const size_t b = evk_bytes(c, evk_digits);
    if (evk_in != evk_out && overlap(evk_in, b, evk_out, b)) HKS_FAIL(HKS_EINVAL, "evk_prepare: partial overlap");
    DevGuard g(c->device);
    return launch_evk_prepare(c, evk_in, evk_out, evk_digits, (cudaStream_t)stream);
}

extern "C" hks_status hks_automorph(const hks_ctx *c, const uint64_t *in, uint32_t nlimbs, uint64_t galois,
                                    uint64_t *out, void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!in || !out || nlimbs == 0) HKS_FAIL(HKS_EINVAL, "automorph: NULL buffer / empty batch");
    if ((st = check_galois(c, galois)) != HKS_OK) return st;
    if (overlap(in, nlimbs * limb_bytes(c), out, nlimbs * limb_bytes(c))) HKS_FAIL(HKS_EINVAL, "automorph: in and out overlap");
    DevGuard g(c->device);
    return launch_automorph(in, out, nlimbs, c->log_n, galois, (cudaStream_t)stream);
}

extern "C" hks_status hks_rotate_hoisted(const hks_ctx *c, const uint64_t *c0, const uint64_t *c1, uint32_t level,
                                         uint32_t nrot, const uint64_t *galois, const uint64_t *const *evk,
                                         uint32_t evk_digits, uint64_t *const *out0, uint64_t *const *out1, void *ws,
                                         void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!c0 || !c1 || !ws || (nrot && (!galois || !evk || !out0 || !out1))) HKS_FAIL(HKS_EINVAL, "rotate_hoisted: NULL argument");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "rotate_hoisted: level %u > L", level);
    if (nrot == 0) return HKS_OK;
    if ((st = check_evk(c, evk_digits, level, "rotate_hoisted")) != HKS_OK) return st;
    const size_t lb = limb_bytes(c), l1 = level + 1, ne = c->ne(level), beta = c->beta(level);
    const size_t wsb = hks_workspace_bytes(c, HKS_OP_ROTATE_HOISTED, level, nrot);
    for (u32 r = 0; r < nrot; r++) {
        if ((st = check_galois(c, galois[r])) != HKS_OK) return st;
        if (!evk[r] || !out0[r] || !out1[r]) HKS_FAIL(HKS_EINVAL, "rotate_hoisted: NULL pointer in arrays");
        if (overlap(out0[r], l1 * lb, c0, l1 * lb) || overlap(out0[r], l1 * lb, c1, l1 * lb) ||
            overlap(out1[r], l1 * lb, c0, l1 * lb) || overlap(out1[r], l1 * lb, c1, l1 * lb) ||
            overlap(out0[r], l1 * lb, ws, wsb) || overlap(out1[r], l1 * lb, ws, wsb) ||
            overlap(out0[r], l1 * lb, out1[r], l1 * lb))
            HKS_FAIL(HKS_EINVAL, "rotate_hoisted: output %u overlaps", r);
    }
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    u64 *coef = (u64 *)ws;
    u64 *ext = coef + l1 * c->n;
    if ((st = modup_core(c, c1, level, ext, coef, s)) != HKS_OK) return st;
    // the rotations split into nb contiguous ranges, one per branch (caller's stream, side streams); a
    // branch takes its range in groups of RB: RB key products (each with its automorphism gather) into RB
    // accumulator pairs, then ONE ModDown over the 2 RB polynomials (large batches per launch)
    // (one branch while profiling; the workspace, sized for rot_branches, holds the single-branch layout too)
    const u32 nb = prof_active() ? 1u : (u32)rot_branches(c, nrot);
    const u32 per = (nrot + nb - 1) / nb;
    const u32 RB = (u32)std::min<size_t>(per, rot_batch(c, level));
    const size_t bw = (size_t)RB * (2 * ne + 2 * c->np + 2 * l1) * c->n;   // words per branch
    SideFork fk(c, s);
    if ((st = fk.fork((int)nb, "rotate_hoisted")) != HKS_OK) return st;
    for (u32 b = 0; b < nb; b++) {
        const cudaStream_t bs = fk.stream((int)b);
        u64 *acc = ext + beta * ne * c->n + b * bw;
        u64 *md = acc + (size_t)RB * 2 * ne * c->n;
        const u32 rend = std::min(nrot, (b + 1) * per);
        for (u32 r0 = b * per; r0 < rend; r0 += RB) {
            const u32 nr = std::min(RB, rend - r0);
            std::vector<u64 *> outs(2 * nr);
            std::vector<const u64 *> adds(2 * nr);
            std::vector<u64> gal(2 * nr);
            for (u32 r = 0; r < nr; r++) {
                if ((st = kip_core(c, ext, c1, evk[r0 + r], level, galois[r0 + r], acc + (size_t)r * 2 * ne * c->n, bs)) !=
                    HKS_OK)
                    return st;
                outs[2 * r] = out0[r0 + r];
                outs[2 * r + 1] = out1[r0 + r];
                adds[2 * r] = c0;
                adds[2 * r + 1] = nullptr;
                gal[2 * r] = galois[r0 + r];
                gal[2 * r + 1] = 1;
            }
            if ((st = moddown_core(c, acc, 2 * nr, level, outs.data(), adds.data(), gal.data(), md, bs, false, nullptr,
                                   evk_prepared(evk_digits))) != HKS_OK)
                return st;
        }
    }
    return fk.join("rotate_hoisted");
}

extern "C" hks_status hks_rotate_hoisted_batch(const hks_ctx *c, uint32_t nct, const uint64_t *const *c0,
                                               const uint64_t *const *c1, uint32_t level, uint32_t nrot,
                                               const uint64_t *galois, const uint64_t *const *evk, uint32_t evk_digits,
                                               uint64_t *const *out0, uint64_t *const *out1, void *ws, void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (nct == 0 || nrot == 0) return HKS_OK;
    if (!c0 || !c1 || !galois || !evk || !out0 || !out1 || !ws) HKS_FAIL(HKS_EINVAL, "rotate_hoisted_batch: NULL argument");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "rotate_hoisted_batch: level %u > L", level);
    if (nct > KIP_MAXCT) HKS_FAIL(HKS_EINVAL, "rotate_hoisted_batch: at most %d ciphertexts per call", KIP_MAXCT);
    const u32 beta = c->beta(level);
    if (beta > 4) HKS_FAIL(HKS_EINVAL, "rotate_hoisted_batch: beta %u > 4", beta);
    if ((st = check_evk(c, evk_digits, level, "rotate_hoisted_batch")) != HKS_OK) return st;
    for (u32 r = 0; r < nrot; r++)
        if (!evk[r]) HKS_FAIL(HKS_EINVAL, "rotate_hoisted_batch: NULL key %u", r);
    for (u32 r = 0; r < nrot; r++)
        if ((st = check_galois(c, galois[r])) != HKS_OK) return st;
    for (u32 i = 0; i < nct * nrot; i++)
        if (!out0[i] || !out1[i]) HKS_FAIL(HKS_EINVAL, "rotate_hoisted_batch: NULL output");
    for (u32 i = 0; i < nct; i++)
        if (!c0[i] || !c1[i]) HKS_FAIL(HKS_EINVAL, "rotate_hoisted_batch: NULL input");
    DevGuard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t N = c->n, l1 = level + 1, ne = c->ne(level), K = c->np;
    u64 *base = (u64 *)ws;
    u64 *coef = base;
    u64 *exts = coef + l1 * N;                          // [nct][beta][ne]
    u64 *accs = exts + (size_t)nct * beta * ne * N;     // [nct][2][ne]
    u64 *md = accs + (size_t)nct * 2 * ne * N;          // ModDown workspace for 2 nct polynomials
    const size_t accw = (size_t)nct * 2 * ne * N, mdw = (size_t)nct * (2 * K + 2 * l1) * N;
    for (u32 i = 0; i < nct; i++)
        if ((st = modup_core(c, c1[i], level, exts + (size_t)i * beta * ne * N, coef, s)) != HKS_OK) return st;
    // the rotations are independent after the ModUps: round-robin over the caller's stream and the
    // context's side streams, each branch with its own accumulators and ModDown workspace
    const int nb = (nrot > 1 && c->side[0] && !prof_active()) ? std::min<int>(1 + hks_ctx::NSIDE, (int)nrot) : 1;
    SideFork fk(c, s);
    if ((st = fk.fork(nb, "rotate_hoisted_batch")) != HKS_OK) return st;
    for (u32 r = 0; r < nrot; r++) {
        const int b = (int)(r % (u32)nb);
        const cudaStream_t bs = fk.stream(b);
        u64 *baccs = b == 0 ? accs : md + mdw + (size_t)(b - 1) * (accw + mdw);
        u64 *bmd = b == 0 ? md : baccs + accw;
        KipMultiArgs a{};
        for (u32 i = 0; i < nct; i++) {
            a.ext[i] = exts + (size_t)i * beta * ne * N;
            a.c1[i] = c1[i];
            a.acc[i] = baccs + (size_t)i * 2 * ne * N;
        }
        a.evk = evk[r];
        a.pc = c->d_pc;
        a.galois = galois[r];
        a.nct = nct;
        a.log_n = c->log_n;
        a.level = level;
        a.nq = c->nq;
        a.np = c->np;
        a.ne = (u32)ne;
        a.nk = c->nq + c->np;
        a.beta = beta;
        a.alpha = c->alpha;
        if ((st = launch_kip_multi(a, bs)) != HKS_OK) return st;
        std::vector<u64 *> outs(2 * nct);
        std::vector<const u64 *> adds(2 * nct);
        std::vector<u64> gal(2 * nct);
        for (u32 i = 0; i < nct; i++) {
            outs[2 * i] = out0[(size_t)i * nrot + r];
            outs[2 * i + 1] = out1[(size_t)i * nrot + r];
            adds[2 * i] = c0[i];
            adds[2 * i + 1] = nullptr;
            gal[2 * i] = galois[r];
            gal[2 * i + 1] = 1;
        }
        if ((st = moddown_core(c, baccs, 2 * nct, level, outs.data(), adds.data(), gal.data(), bmd, bs, false, nullptr,
                               evk_prepared(evk_digits))) != HKS_OK)
            return st;
    }
    return fk.join("rotate_hoisted_batch");
}

extern "C" size_t hks_rotate_hoisted_batch_workspace_bytes(const hks_ctx *c, uint32_t nct, uint32_t level) {
    if (!c || level > c->L() || nct == 0) return 0;
    const size_t lb = limb_bytes(c), l1 = level + 1, ne = c->ne(level), K = c->np, beta = c->beta(level);
    // coef, ModUp outputs, then per branch (caller's stream + side streams) accumulators and ModDown workspace
    return (l1 + nct * beta * ne + (1 + hks_ctx::NSIDE) * (nct * 2 * ne + nct * (2 * K + 2 * l1))) * lb;
}

// ------------------------------------------------------------------------------------------------
// BSGS linear transform

namespace {
// chunks of WS_MAXT terms; chunks after the first accumulate into out
hks_status wsum_core(const hks_ctx *c, u32 nterm, const uint64_t *const *w, const uint64_t *const *x0,
                     const uint64_t *const *x1, u32 level, u64 *out0, u64 *out1, cudaStream_t s) {
    for (u32 j0 = 0; j0 < nterm; j0 += WS_MAXT) {
        WsumArgs a{};
        a.nterm = std::min<u32>(WS_MAXT, nterm - j0);
        for (u32 j = 0; j < a.nterm; j++) {
            a.w[j] = w[j0 + j];
            a.x0[j] = x0[j0 + j];
            a.x1[j] = x1[j0 + j];
        }
        a.out0 = out0;
        a.out1 = out1;
        a.pc = c->d_pc;
        a.nlimbs = level + 1;
        a.log_n = c->log_n;
        a.accumulate = j0 > 0;
        hks_status st = launch_pt_wsum(a, s);
        if (st != HKS_OK) return st;
    }
    return HKS_OK;
}
}  // namespace

extern "C" hks_status hks_pt_weighted_sum(const hks_ctx *c, uint32_t nterm, const uint64_t *const *w,
                                          const uint64_t *const *x0, const uint64_t *const *x1, uint32_t level,
                                          uint64_t *out0, uint64_t *out1, void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!w || !x0 || !x1 || !out0 || !out1 || nterm == 0) HKS_FAIL(HKS_EINVAL, "pt_weighted_sum: NULL argument / no term");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "pt_weighted_sum: level %u > L", level);
    const size_t sz = (level + 1) * limb_bytes(c);
    if (overlap(out0, sz, out1, sz)) HKS_FAIL(HKS_EINVAL, "pt_weighted_sum: outputs overlap");
    for (u32 j = 0; j < nterm; j++) {
        if (!w[j] || !x0[j] || !x1[j]) HKS_FAIL(HKS_EINVAL, "pt_weighted_sum: NULL term %u", j);
        const void *ins[3] = {w[j], x0[j], x1[j]};
        for (const void *p : ins)
            if (overlap(p, sz, out0, sz) || overlap(p, sz, out1, sz))
                HKS_FAIL(HKS_EINVAL, "pt_weighted_sum: an output overlaps term %u", j);
    }
    DevGuard g(c->device);
    return wsum_core(c, nterm, w, x0, x1, level, out0, out1, (cudaStream_t)stream);
}

extern "C" size_t hks_linear_transform_workspace_bytes(const hks_ctx *c, uint32_t level, uint32_t n1) {
    if (!c || level > c->L() || n1 == 0) return 0;
    const size_t lb = limb_bytes(c), l1 = level + 1;
    const size_t rot = std::max(hks_workspace_bytes(c, HKS_OP_ROTATE_HOISTED, level, n1 > 1 ? n1 - 1 : 1),
                                hks_workspace_bytes(c, HKS_OP_ROTATE_HOISTED, level, 1));
    const size_t rot1 = hks_workspace_bytes(c, HKS_OP_ROTATE_HOISTED, level, 1);
    // baby ciphertexts, inner, rotated inner, rotations; per side branch: inner, rotated, accumulator, rotation
    return (2 * (size_t)(n1 - 1) + 4) * l1 * lb + rot + hks_ctx::NSIDE * (6 * l1 * lb + rot1);
}

extern "C" hks_status hks_linear_transform(const hks_ctx *c, const uint64_t *c0, const uint64_t *c1, uint32_t level,
                                           uint32_t n1, uint32_t n2, const uint64_t *baby_galois,
                                           const uint64_t *const *baby_evk, const uint64_t *giant_galois,
                                           const uint64_t *const *giant_evk, uint32_t evk_digits,
                                           const uint64_t *const *pt, uint64_t *out0, uint64_t *out1, void *ws,
                                           void *stream) {
    hks_status st = check_ctx(c);
    if (st != HKS_OK) return st;
    if (!c0 || !c1 || !pt || !out0 || !out1 || !ws) HKS_FAIL(HKS_EINVAL, "linear_transform: NULL argument");
    if (n1 == 0 || n2 == 0 || n1 > 1024 || n2 > 1024) HKS_FAIL(HKS_EINVAL, "linear_transform: n1, n2 must be in [1, 1024]");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "linear_transform: level %u > L", level);
    if ((n1 > 1 && (!baby_galois || !baby_evk)) || (n2 > 1 && (!giant_galois || !giant_evk)))
        HKS_FAIL(HKS_EINVAL, "linear_transform: missing rotation keys");
    for (u32 k = 0; k + 1 < n2; k++)
        if ((st = check_galois(c, giant_galois[k])) != HKS_OK) return st;
    if ((n1 > 1 || n2 > 1) && (st = check_evk(c, evk_digits, level, "linear_transform")) != HKS_OK) return st;
    for (u32 k = 0; k < n1 * n2; k++)
        if (!pt[k]) HKS_FAIL(HKS_EINVAL, "linear_transform: NULL diagonal %u", k);
    const size_t lb = limb_bytes(c), l1 = level + 1, sz = l1 * lb;
    const size_t wsb = hks_linear_transform_workspace_bytes(c, level, n1);
    if (overlap(out0, sz, c0, sz) || overlap(out0, sz, c1, sz) || overlap(out1, sz, c0, sz) ||
        overlap(out1, sz, c1, sz) || overlap(out0, sz, out1, sz) || overlap(out0, sz, ws, wsb) ||
        overlap(out1, sz, ws, wsb))
        HKS_FAIL(HKS_EINVAL, "linear_transform: outputs overlap an input or ws");
    cudaStream_t s = (cudaStream_t)stream;
    DevGuard g(c->device);
    u64 *base = (u64 *)ws;
    const size_t lw = l1 * c->n;   // words per polynomial
    // ciphertext j (j = 0: the input; j >= 1: baby rotation j) halves
    std::vector<const u64 *> x0(n1), x1(n1);
    std::vector<u64 *> b0(n1), b1(n1);
    x0[0] = c0;
    x1[0] = c1;
    for (u32 j = 1; j < n1; j++) {
        b0[j] = base + (2 * (size_t)(j - 1)) * lw;
        b1[j] = b0[j] + lw;
        x0[j] = b0[j];
        x1[j] = b1[j];
    }
    const size_t rotb = hks_workspace_bytes(c, HKS_OP_ROTATE_HOISTED, level, n1 > 1 ? n1 - 1 : 1);
    const size_t rot = std::max(rotb, hks_workspace_bytes(c, HKS_OP_ROTATE_HOISTED, level, 1));
    const size_t rot1w = hks_workspace_bytes(c, HKS_OP_ROTATE_HOISTED, level, 1) / 8;
    // branch 0 = the caller's stream (accumulates into out), branch b >= 1 = side stream b - 1 (own inner,
    // rotated and accumulator buffers and rotation workspace, summed into out after the join)
    struct Branch { u64 *i0, *i1, *r0, *r1, *a0, *a1, *rws; cudaStream_t s; bool first; };
    Branch br[1 + hks_ctx::NSIDE];
    {
        u64 *at = base + 2 * (size_t)(n1 - 1) * lw;
        br[0] = {at, at + lw, at + 2 * lw, at + 3 * lw, out0, out1, at + 4 * lw, s, false};
        at += 4 * lw + rot / 8;
        for (int b = 1; b <= hks_ctx::NSIDE; b++) {
            br[b] = {at, at + lw, at + 2 * lw, at + 3 * lw, at + 4 * lw, at + 5 * lw, at + 6 * lw, c->side[b - 1], true};
            at += 6 * lw + rot1w;
        }
    }
    // baby steps: one ModUp shared by the n1 - 1 rotations (hoisted)
    if (n1 > 1 && (st = hks_rotate_hoisted(c, c0, c1, level, n1 - 1, baby_galois, baby_evk, evk_digits, b0.data() + 1,
                                           b1.data() + 1, br[0].rws, stream)) != HKS_OK)
        return st;
    // giant steps: I_i = sum_j pt[i n1 + j] ct_j (fused weighted sum), out += Rot_{g_i}(I_i).  The giant
    // steps are independent: with more than two of them, steps i = 1, 2, ... go round-robin to the caller's
    // stream and the side streams (modular sums are exact, so the order of the additions does not matter)
    if ((st = wsum_core(c, n1, pt, x0.data(), x1.data(), level, out0, out1, s)) != HKS_OK) return st;
    const int nb = (n2 > 2 && c->side[0] && !prof_active()) ? std::min<int>(1 + hks_ctx::NSIDE, (int)n2 - 1) : 1;
    SideFork fk(c, s);
    if ((st = fk.fork(nb, "linear_transform")) != HKS_OK) return st;
    for (u32 i = 1; i < n2; i++) {
        Branch &B = br[(i - 1) % nb];
        if ((st = wsum_core(c, n1, pt + (size_t)i * n1, x0.data(), x1.data(), level, B.i0, B.i1, B.s)) != HKS_OK)
            return st;
        u64 *o0 = B.first ? B.a0 : B.r0, *o1 = B.first ? B.a1 : B.r1;
        if ((st = hks_rotate_hoisted(c, B.i0, B.i1, level, 1, giant_galois + (i - 1), giant_evk + (i - 1), evk_digits,
                                     &o0, &o1, B.rws, B.s)) != HKS_OK)
            return st;
        if (!B.first && (st = launch_add_ct(B.r0, B.r1, B.a0, B.a1, level + 1, c->log_n, c->d_pc, B.s)) != HKS_OK)
            return st;
        B.first = false;
    }
    if ((st = fk.join("linear_transform")) != HKS_OK) return st;
    for (int b = 1; b < nb; b++)
        if ((st = launch_add_ct(br[b].a0, br[b].a1, out0, out1, level + 1, c->log_n, c->d_pc, s)) != HKS_OK) return st;
    return HKS_OK;
}
