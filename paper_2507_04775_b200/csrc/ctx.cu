// ctx.cu -- context creation: validation and one-time precomputation (§3.5).
//
// The library's own host number theory (independent of oracle/): Montgomery-free u128 arithmetic,
// deterministic Miller-Rabin, the minimal primitive 2N-th root, bit-reversed twiddle tables with
// Shoup companions, the Eq. 1 ModUp constants per (level, digit), and the ModDown constants.
// Unlike the paper's singleton a context is an ordinary immutable handle; the
// per-prime scalars every thread needs travel in kernel parameters / read-only loads instead of
// a 64 KB __constant__ bank.
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <thread>

#include <atomic>

#include "internal.h"

typedef unsigned __int128 u128;

static thread_local char g_err[512] = "";

void hks_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

extern "C" const char *hks_last_error(void) { return g_err; }

namespace {

u64 mul_mod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }

u64 pow_mod(u64 a, u64 e, u64 m) {
    u64 r = 1 % m;
    a %= m;
    for (; e; e >>= 1, a = mul_mod(a, a, m))
        if (e & 1) r = mul_mod(r, a, m);
    return r;
}

u64 inv_mod(u64 a, u64 m) { return pow_mod(a, m - 2, m); }   // m prime

bool is_prime64(u64 n) {
    if (n < 2) return false;
    static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (u64 s : small)
        if (n % s == 0) return n == s;
    u64 d = n - 1;
    int r = 0;
    while (!(d & 1)) d >>= 1, r++;
    for (u64 a : small) {
        u64 x = pow_mod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < r && comp; i++) {
            x = mul_mod(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}

// SURVEY.md §8(c) reading 1: the smallest x with x^N = -1 (mod m).  Every such x is psi0^k, k odd.
u64 minimal_psi(u64 m, u32 n) {
    u64 psi0 = 0;
    for (u64 g = 2;; g++) {
        u64 c = pow_mod(g, (m - 1) / (2 * (u64)n), m);
        if (pow_mod(c, n, m) == m - 1) { psi0 = c; break; }
    }
    u64 step = mul_mod(psi0, psi0, m), cur = psi0, best = psi0;
    for (u32 k = 0; k < n; k++) {
        best = std::min(best, cur);
        cur = mul_mod(cur, step, m);
    }
    return best;
}

u64 shoup_of(u64 w, u64 m) { return (u64)(((u128)w << 64) / m); }

ulonglong2 sh(u64 w, u64 m) { return make_ulonglong2(w, shoup_of(w, m)); }

uint2 split(u64 v) { return make_uint2((u32)(v & 0x3fffffffu), (u32)(v >> 30)); }

u32 bitrev(u32 x, u32 bits) {
    u32 r = 0;
    for (u32 i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}

template <typename T>
hks_status upload(T **dptr, const std::vector<T> &h) {
    if (h.empty()) { *dptr = nullptr; return HKS_OK; }
    cudaError_t e = cudaMalloc((void **)dptr, h.size() * sizeof(T));
    if (e != cudaSuccess) HKS_FAIL(HKS_ENOMEM, "cudaMalloc(%zu): %s", h.size() * sizeof(T), cudaGetErrorString(e));
    e = cudaMemcpy(*dptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) HKS_FAIL(HKS_ECUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
    return HKS_OK;
}

void free_tables(hks_ctx *c) {
    void *ptrs[] = {c->d_pc, c->d_tw_all, c->d_ninv,
                    c->d_mu_scale, c->d_mu_mat, c->d_md_scale, c->d_md_mat, c->d_pinv, c->d_mu_matf, c->d_md_matf, c->d_mu_mats, c->d_md_mats, c->d_mu_matb, c->d_md_matb, c->d_mu_img, c->d_md_img, c->d_ntt_img_fwd, c->d_ntt_img_inv,
                    c->d_qmod, c->d_qlinv, c->d_mdp_mat, c->d_mdp_mats, c->d_mdp_matf, c->d_mdp_matb, c->d_mdp_img};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < hks_ctx::NSIDE; i++) {
        if (c->side[i]) cudaStreamDestroy(c->side[i]);
        if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
}

// Twiddle tables of one prime.  psi_brv[k] = psi^brv_logN(k) ("precomputing the
// twiddle factors ... Shoup constants are also precomputed").  Column table = psi_brv[0..R);
// row table of row r at heap index k = 2^s + i:  psi_brv[(R + r) 2^s + i].
void twiddles(u64 m, u64 root, u32 log_n, u32 log_r, u32 log_c, ulonglong2 *col, ulonglong2 *row) {
    const u32 n = 1u << log_n, R = 1u << log_r, C = 1u << log_c;
    std::vector<u64> pw(n);
    u64 x = 1;
    for (u32 e = 0; e < n; e++) { pw[e] = x; x = mul_mod(x, root, m); }
    auto psi_brv = [&](u32 k) { return pw[bitrev(k, log_n)]; };
    for (u32 k = 0; k < R; k++) col[k] = sh(psi_brv(k), m);
    for (u32 r = 0; r < R; r++) {
        row[(size_t)r * C] = make_ulonglong2(0, 0);
        for (u32 s = 0; (1u << s) < C; s++)
            for (u32 i = 0; i < (1u << s); i++)
                row[(size_t)r * C + (1u << s) + i] = sh(psi_brv(((R + r) << s) + i), m);
    }
}

}  // namespace

// Byte-column words of a base-conversion matrix entry v = [qhat]_t (tensor-pipe BConv, k_bconv_mma):
// m_a = 2^(8a) v mod t for a = 0..7, and word c (c = 0..7) holds byte c of m_a in its byte a.  Then
// for any y = sum_a y_a 2^(8a):  sum_a y_a m_a = sum_c 2^(8c) sum_a y_a byte_c(m_a) == y v (mod t).
void push_bytecols(std::vector<u64> &out, u64 v, u64 t) {
    u64 m[8];
    m[0] = v % t;
    for (int a = 1; a < 8; a++) m[a] = (u64)(((u128)m[a - 1] << 8) % t);
    for (int c = 0; c < 8; c++) {
        u64 w = 0;
        for (int a = 0; a < 8; a++) w |= ((m[a] >> (8 * c)) & 0xffull) << (8 * a);
        out.push_back(w);
    }
}


// B-operand image of k_bconv_tc (internal.h bconv_img_words) from byte-column words [nsrc][ntg][8]:
// image word (t, kc, c, h) = word (2kc + h, t, c), zero past the sources.
void bconv_image(const u64 *matb, u32 nsrc, u32 ntg, std::vector<u64> &out) {
    const u32 nch = bconv_img_words(nsrc) / 16;
    for (u32 t = 0; t < ntg; t++)
        for (u32 kc = 0; kc < nch; kc++)
            for (u32 cc = 0; cc < 8; cc++)
                for (u32 hh = 0; hh < 2; hh++) {
                    const u32 i = 2 * kc + hh;
                    out.push_back(i < nsrc ? matb[((size_t)i * ntg + t) * 8 + cc] : 0);
                }
}

extern "C" hks_status hks_ctx_create(uint32_t log_n, const uint64_t *q, uint32_t num_q, const uint64_t *p,
                                     uint32_t num_p, uint32_t dnum, int device, hks_ctx **out) {
    if (!out || !q || !p) HKS_FAIL(HKS_EINVAL, "ctx_create: NULL argument");
    *out = nullptr;
    if (log_n < 10 || log_n > 17) HKS_FAIL(HKS_ERANGE, "ctx_create: log_n %u outside [10, 17]", log_n);
    if (num_q < 1 || num_p < 1) HKS_FAIL(HKS_EINVAL, "ctx_create: need at least one q and one p");
    if (dnum < 1 || dnum > num_q) HKS_FAIL(HKS_ERANGE, "ctx_create: dnum %u outside [1, %u]", dnum, num_q);
    if (num_q + num_p > 1024) HKS_FAIL(HKS_ERANGE, "ctx_create: too many moduli");
    const u32 alpha = (num_q + dnum - 1) / dnum;
    if (alpha > BC_MAXSRC) HKS_FAIL(HKS_ERANGE, "ctx_create: alpha = ceil((L+1)/dnum) = %u > %d unsupported", alpha, BC_MAXSRC);
    if (num_p > BC_MAXSRC) HKS_FAIL(HKS_ERANGE, "ctx_create: K = %u > %d unsupported", num_p, BC_MAXSRC);
    const u32 n = 1u << log_n;
    std::vector<u64> primes(q, q + num_q);
    primes.insert(primes.end(), p, p + num_p);
    for (size_t i = 0; i < primes.size(); i++) {
        u64 m = primes[i];
        if (m >= (1ull << 60)) HKS_FAIL(HKS_ERANGE, "ctx_create: modulus %zu = %llu >= 2^60", i, (unsigned long long)m);
        if (!is_prime64(m)) HKS_FAIL(HKS_ENOTPRIME, "ctx_create: modulus %zu = %llu is not prime", i, (unsigned long long)m);
        if ((m - 1) % (2 * (u64)n)) HKS_FAIL(HKS_ENOTNTT, "ctx_create: modulus %zu = %llu is not 1 mod 2N", i, (unsigned long long)m);
        for (size_t j = 0; j < i; j++)
            if (primes[j] == m) HKS_FAIL(HKS_EDUP, "ctx_create: modulus %llu repeated", (unsigned long long)m);
    }
    if (device >= 0) {
        int cnt = 0;
        if (cudaGetDeviceCount(&cnt) != cudaSuccess || device >= cnt)
            HKS_FAIL(HKS_EDEVICE, "ctx_create: CUDA device %d not available", device);
    }

    hks_ctx *c = new hks_ctx();
    c->log_n = log_n;
    c->n = n;
    c->log_r = (log_n + 1) / 2;
    c->log_c = log_n / 2;
    c->nq = num_q;
    c->np = num_p;
    c->dnum = dnum;
    c->alpha = alpha;
    c->device = device;
    c->primes = primes;
    const u32 nm = (u32)primes.size();
    c->psi.resize(nm);
    {
        std::vector<std::thread> th;
        u32 nt = std::max(1u, std::min(nm, std::thread::hardware_concurrency()));
        for (u32 w = 0; w < nt; w++)
            th.emplace_back([&, w] {
                for (u32 i = w; i < nm; i += nt) c->psi[i] = minimal_psi(primes[i], n);
            });
        for (auto &t : th) t.join();
    }
    if (device < 0) { *out = c; return HKS_OK; }

    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) { delete c; HKS_FAIL(HKS_EDEVICE, "ctx_create: cudaSetDevice(%d) failed", device); }

    const u32 R = 1u << c->log_r, L = num_q - 1;
    std::vector<PrimeConst> pc(nm);
    std::vector<ulonglong2> ninv(nm);
    for (u32 i = 0; i < nm; i++) {
        u64 m = primes[i];
        u64 r64 = (u64)(((u128)1 << 64) % m);
        const u128 mu80 = ((u128)1 << 80) / m;   // used only when every prime > 2^49 (then < 2^31)
        pc[i] = PrimeConst{m, r64, shoup_of(r64, m), (u64)(~0ull / m), mu80 >> 64 ? 0 : (u64)mu80};
        if (m >> 49 == 0) c->all_big = false;   // the byte-sum reduction needs p > 2^49
        ninv[i] = sh(inv_mod(n % m, m), m);
    }
    // one_p = floor(2^64 / m) = floor((2^64 - 1) / m) since m does not divide 2^64.
    std::vector<ulonglong2> tcf((size_t)nm * R), trf((size_t)nm * n), tci((size_t)nm * R), tri((size_t)nm * n);
    {
        std::vector<std::thread> th;
        u32 nt = std::max(1u, std::min(nm, std::thread::hardware_concurrency()));
        for (u32 w = 0; w < nt; w++)
            th.emplace_back([&, w] {
                for (u32 i = w; i < nm; i += nt) {
                    u64 m = primes[i];
                    twiddles(m, c->psi[i], log_n, c->log_r, c->log_c, &tcf[(size_t)i * R], &trf[(size_t)i * n]);
                    twiddles(m, inv_mod(c->psi[i], m), log_n, c->log_r, c->log_c, &tci[(size_t)i * R], &tri[(size_t)i * n]);
                }
            });
        for (auto &t : th) t.join();
    }

    // ModUp constants (Eq. 1) per level l and digit j: scale N^-1 [qhat_{j,i}]^-1 mod q_i for the
    // digit's active limbs, matrix [qhat_{j,i}]_t for targets t in (Q_l \ digit j) u P.
    std::vector<ulonglong2> mu_scale;
    std::vector<uint2> mu_mat;
    std::vector<u64> mu_matb;
    c->mu_scale_off.resize(num_q);
    c->mu_mat_off.assign((size_t)num_q * dnum, 0);
    for (u32 lv = 0; lv <= L; lv++) {
        c->mu_scale_off[lv] = mu_scale.size();
        u32 beta = c->beta(lv);
        for (u32 i = 0; i <= lv; i++) {
            u32 j = i / alpha, lo = c->digit_lo(j), hi = c->digit_hi(lv, j);
            u64 m = primes[i], h = 1;
            for (u32 k = lo; k < hi; k++)
                if (k != i) h = mul_mod(h, primes[k] % m, m);
            mu_scale.push_back(sh(mul_mod(inv_mod(h, m), inv_mod(n % m, m), m), m));
        }
        for (u32 j = 0; j < beta; j++) {
            c->mu_mat_off[(size_t)lv * dnum + j] = mu_mat.size();
            u32 lo = c->digit_lo(j), hi = c->digit_hi(lv, j);
            for (u32 i = lo; i < hi; i++)
                for (u32 t = 0; t < c->ne(lv); t++) {
                    if (t >= lo && t < hi) continue;
                    u64 m = primes[c->ext_prime(lv, t)], h = 1;
                    for (u32 k = lo; k < hi; k++)
                        if (k != i) h = mul_mod(h, primes[k] % m, m);
                    mu_mat.push_back(split(h));
                    push_bytecols(mu_matb, h, m);
                }
        }
    }
    // ModDown constants: scale N^-1 [phat_k]^-1 mod p_k, matrix [phat_k]_{q_i} [K][L+1], P^-1 mod q_i.
    std::vector<ulonglong2> md_scale(num_p), pinv(num_q);
    std::vector<uint2> md_mat((size_t)num_p * num_q);
    std::vector<u64> md_matb((size_t)num_p * num_q * 8);
    for (u32 k = 0; k < num_p; k++) {
        u64 m = p[k], h = 1;
        for (u32 o = 0; o < num_p; o++)
            if (o != k) h = mul_mod(h, p[o] % m, m);
        md_scale[k] = sh(mul_mod(inv_mod(h, m), inv_mod(n % m, m), m), m);
        for (u32 i = 0; i < num_q; i++) {
            u64 qi = q[i], hv = 1;
            for (u32 o = 0; o < num_p; o++)
                if (o != k) hv = mul_mod(hv, p[o] % qi, qi);
            md_mat[(size_t)k * num_q + i] = split(hv);
            std::vector<u64> w;
            push_bytecols(w, hv, qi);
            std::copy(w.begin(), w.end(), md_matb.begin() + ((size_t)k * num_q + i) * 8);
        }
    }
    for (u32 i = 0; i < num_q; i++) {
        u64 qi = q[i], P = 1;
        for (u32 k = 0; k < num_p; k++) P = mul_mod(P, p[k] % qi, qi);
        pinv[i] = sh(inv_mod(P, qi), qi);
    }
    // hks_evk_prepare keys: ModDown matrix entries times P^-1 mod q_i (the epilogue then skips its P^-1 product)
    std::vector<uint2> mdp_mat(md_mat.size());
    std::vector<u64> mdp_matb(md_matb.size());
    for (u32 k = 0; k < num_p; k++)
        for (u32 i = 0; i < num_q; i++) {
            const size_t e = (size_t)k * num_q + i;
            const u64 hv = (u64)md_mat[e].x | ((u64)md_mat[e].y << 30);
            const u64 hvp = mul_mod(hv, pinv[i].x, q[i]);
            mdp_mat[e] = split(hvp);
            std::vector<u64> w;
            push_bytecols(w, hvp, q[i]);
            std::copy(w.begin(), w.end(), mdp_matb.begin() + e * 8);
        }

    // Rescale constants: q_j mod q_i (centered SwitchModulo from q_j into q_i) and
    // q_j^-1 mod q_i (Shoup), row j = the dropped limb, [L+1][L+1]; diagonal unused.
    std::vector<u64> qmod((size_t)num_q * num_q, 0);
    std::vector<ulonglong2> qlinv((size_t)num_q * num_q, make_ulonglong2(0, 0));
    for (u32 j = 0; j < num_q; j++)
        for (u32 i = 0; i < num_q; i++) {
            if (i == j) continue;
            qmod[(size_t)j * num_q + i] = q[j] % q[i];
            qlinv[(size_t)j * num_q + i] = sh(inv_mod(q[j] % q[i], q[i]), q[i]);
        }

    // the same matrices as exact 20-bit limbs in doubles (FP64-pipe part of k_bconv_fp)
    auto limbs20 = [](const std::vector<uint2> &m) {
        std::vector<double> f(m.size() * 3);
        for (size_t i = 0; i < m.size(); i++) {
            const u64 v = (u64)m[i].x | ((u64)m[i].y << 30);
            f[3 * i + 0] = (double)(v & 0xfffff);
            f[3 * i + 1] = (double)((v >> 20) & 0xfffff);
            f[3 * i + 2] = (double)(v >> 40);
        }
        return f;
    };
    std::vector<double> mu_matf = limbs20(mu_mat), md_matf = limbs20(md_mat), mdp_matf = limbs20(mdp_mat);
    auto sums = [](const std::vector<uint2> &m) {
        std::vector<u32> f(m.size());
        for (size_t i = 0; i < m.size(); i++) f[i] = m[i].x + m[i].y;
        return f;
    };
    std::vector<u32> mu_mats = sums(mu_mat), md_mats = sums(md_mat), mdp_mats = sums(mdp_mat);

    // k_bconv_tc B-operand images (internal.h bconv_img_words): image word (t, kc, c, h) = matb word
    // (2kc + h, t, c), zero past the sources
    auto image = bconv_image;
    std::vector<u64> mu_img, md_img, mdp_img;
    // Column-pass tables of the tensor-core NTT (log N = 16 only; R = C = 256; ntt_tc.cu).  The butterfly
    // stages of the pass (the same twiddles as k_ntt) are applied to unit vectors, giving the 16 x 16
    // matrices of its two rounds: forward = W_A (stages 0-3, any stride-16 class) then W_B[b] (stages 4-7,
    // block b) = W_B[0] diag(d_b); inverse = W'_B[b] (GS stages 7-4) = diag(f_b) W'_B[0] then W'_A (GS
    // stages 3-0).  Per prime and direction: image of round 1 (W_A / W'_B[0]), image of round 2
    // (W_B[0] / W'_A), and the twist between the rounds as Shoup pairs tw[v][o] for round-1 vector class v
    // and output o (forward d_o[v], inverse f_v[o]).
    std::vector<u64> ntt_img_fwd, ntt_img_inv;
    if (log_n == 16) {
        ntt_img_fwd.reserve((size_t)nm * NTT16_TAB);
        ntt_img_inv.reserve((size_t)nm * NTT16_TAB);
        for (u32 pi = 0; pi < nm; pi++) {
            const u64 m = primes[pi];
            const ulonglong2 *twf = &tcf[(size_t)pi * R], *twi = &tci[(size_t)pi * R];
            // stages s_from .. s_to of the 256-row column transform on a unit vector at `row`
            auto run = [&](bool fwd, int s_from, int s_to, u32 row, std::vector<u64> &v) {
                v.assign(R, 0);
                v[row] = 1;
                const int step = fwd ? 1 : -1;
                for (int st = s_from;; st += step) {
                    const u32 mm = 1u << st, t = R >> (st + 1);
                    for (u32 i = 0; i < mm; i++) {
                        const u64 w = fwd ? twf[mm + i].x : twi[mm + i].x;
                        for (u32 jj = i * 2 * t; jj < i * 2 * t + t; jj++) {
                            const u64 X = v[jj], Y = v[jj + t];
                            if (fwd) {
                                const u64 wy = mul_mod(Y, w, m);
                                v[jj] = (X + wy) % m;
                                v[jj + t] = (X + m - wy) % m;
                            } else {
                                v[jj] = (X + Y) % m;
                                v[jj + t] = mul_mod((X + m - Y) % m, w, m);
                            }
                        }
                    }
                    if (st == s_to) break;
                }
            };
            // W[k'][k]: rows {base + str k} -> {base + str k'}
            auto matrix = [&](bool fwd, int s_from, int s_to, u32 base, u32 str) {
                std::vector<u64> W(256), v;
                for (u32 k = 0; k < 16; k++) {
                    run(fwd, s_from, s_to, base + str * k, v);
                    for (u32 kk = 0; kk < 16; kk++) W[kk * 16 + k] = v[base + str * kk];
                }
                return W;
            };
            auto emit_image = [&](const std::vector<u64> &W, std::vector<u64> &out) {
                std::vector<u64> words((size_t)16 * 16 * 8), w8;   // matb layout [k][k'][c]
                for (u32 k = 0; k < 16; k++)
                    for (u32 kk = 0; kk < 16; kk++) {
                        w8.clear();
                        push_bytecols(w8, W[kk * 16 + k], m);
                        std::copy(w8.begin(), w8.end(), words.begin() + ((size_t)k * 16 + kk) * 8);
                    }
                image(words.data(), 16, 16, out);
            };
            for (int dir = 0; dir < 2; dir++) {
                const bool fwd = dir == 0;
                std::vector<u64> &out = fwd ? ntt_img_fwd : ntt_img_inv;
                const std::vector<u64> W1 = fwd ? matrix(true, 0, 3, 0, 16) : matrix(false, 7, 4, 0, 1);
                const std::vector<u64> W2 = fwd ? matrix(true, 4, 7, 0, 1) : matrix(false, 3, 0, 0, 16);
                emit_image(W1, out);
                emit_image(W2, out);
                std::vector<std::vector<u64>> Wb(16);
                for (u32 b = 0; b < 16; b++) Wb[b] = fwd ? matrix(true, 4, 7, 16 * b, 1) : matrix(false, 7, 4, 16 * b, 1);
                for (u32 v = 0; v < 16; v++)
                    for (u32 o = 0; o < 16; o++) {
                        // forward: column v of W_B[o] over column v of W_B[0]; inverse: row o of W'_B[v]
                        // over row o of W'_B[0] (entries are products of roots of unity, never 0)
                        const u64 num = fwd ? Wb[o][0 * 16 + v] : Wb[v][o * 16 + 0];
                        const u64 den = fwd ? W2[0 * 16 + v] : W1[o * 16 + 0];
                        const u64 tw = mul_mod(num, inv_mod(den, m), m);
                        out.push_back(tw);
                        out.push_back(shoup_of(tw, m));
                    }
            }
        }
    }
    c->mu_img_off.assign((size_t)num_q * dnum, 0);
    for (u32 lv = 0; lv <= L; lv++)
        for (u32 j = 0; j < c->beta(lv); j++) {
            const u32 lo = c->digit_lo(j), hi = c->digit_hi(lv, j), ntg = c->ne(lv) - (hi - lo);
            c->mu_img_off[(size_t)lv * dnum + j] = mu_img.size();
            image(mu_matb.data() + 8 * c->mu_mat_off[(size_t)lv * dnum + j], hi - lo, ntg, mu_img);
        }
    image(md_matb.data(), num_p, num_q, md_img);
    image(mdp_matb.data(), num_p, num_q, mdp_img);

    hks_status st = HKS_OK;
#define UP(dst, src) if (st == HKS_OK) st = upload(&c->dst, src)
    UP(d_pc, pc);
    UP(d_ninv, ninv);
    {
        // the four twiddle tables in one allocation, so that one L2 access-policy window covers them
        std::vector<ulonglong2> all;
        all.reserve(tcf.size() + trf.size() + tci.size() + tri.size());
        for (const auto *v : {&tcf, &trf, &tci, &tri}) all.insert(all.end(), v->begin(), v->end());
        UP(d_tw_all, all);
        if (st == HKS_OK) {
            c->d_tw_col_fwd = c->d_tw_all;
            c->d_tw_row_fwd = c->d_tw_col_fwd + tcf.size();
            c->d_tw_col_inv = c->d_tw_row_fwd + trf.size();
            c->d_tw_row_inv = c->d_tw_col_inv + tci.size();
            const size_t bytes = all.size() * sizeof(ulonglong2);
            int maxp = 0, maxw = 0;
            if (HKS_TW_PERSIST && cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device) == cudaSuccess &&
                cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, device) == cudaSuccess && maxp > 0 &&
                maxw > 0) {
                size_t cur = 0;
                cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
                if (cur < (size_t)maxp) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp);
                cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
                // HKS_TW_PERSIST == 2: only the inverse tables (the c1 INTT's per-row table is the 3x re-read)
                const size_t off = HKS_TW_PERSIST == 2 ? (size_t)(c->d_tw_col_inv - c->d_tw_all) : 0;
                c->tw_win.base_ptr = c->d_tw_all + off;
                c->tw_win.num_bytes = std::min(bytes - off * sizeof(ulonglong2), (size_t)maxw);
                c->tw_win.hitRatio = (float)std::min(1.0, (double)cur / (double)c->tw_win.num_bytes);
                c->tw_win.hitProp = cudaAccessPropertyPersisting;
                c->tw_win.missProp = cudaAccessPropertyStreaming;
                cudaGetLastError();
            }
        }
    }
    UP(d_mu_scale, mu_scale);
    UP(d_mu_mat, mu_mat);
    UP(d_md_scale, md_scale);
    UP(d_md_mat, md_mat);
    UP(d_pinv, pinv);
    UP(d_mdp_mat, mdp_mat);
    UP(d_mdp_mats, mdp_mats);
    UP(d_mdp_img, mdp_img);
    if (HKS_EXPERIMENTAL) {   // tables of the FP64-assisted and warp-IMMA base conversions
        UP(d_mu_matf, mu_matf);
        UP(d_md_matf, md_matf);
        UP(d_mu_matb, mu_matb);
        UP(d_md_matb, md_matb);
        UP(d_mdp_matf, mdp_matf);
        UP(d_mdp_matb, mdp_matb);
    }
    UP(d_mu_mats, mu_mats);
    UP(d_mu_img, mu_img);
    UP(d_md_img, md_img);
    UP(d_ntt_img_fwd, ntt_img_fwd);
    UP(d_ntt_img_inv, ntt_img_inv);
    UP(d_md_mats, md_mats);
    UP(d_qmod, qmod);
    UP(d_qlinv, qlinv);
#undef UP
    for (int i = 0; i < hks_ctx::NSIDE && st == HKS_OK; i++) {
        if (cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming) != cudaSuccess)
            st = HKS_ECUDA;
    }
    if (st == HKS_OK && cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess) st = HKS_ECUDA;
    cudaSetDevice(prev);
    if (st != HKS_OK) {
        free_tables(c);
        delete c;
        return st;
    }
    *out = c;
    return HKS_OK;
}

extern "C" void hks_ctx_destroy(hks_ctx *c) {
    if (!c) return;
    if (c->device >= 0) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(c->device);
        free_tables(c);
        cudaSetDevice(prev);
    }
    delete c;
}

extern "C" hks_status hks_ctx_query(const hks_ctx *c, uint32_t level, hks_info *out) {
    if (!c || !out) HKS_FAIL(HKS_EINVAL, "ctx_query: NULL argument");
    if (level > c->L()) HKS_FAIL(HKS_EINVAL, "ctx_query: level %u > L = %u", level, c->L());
    *out = hks_info{};
    out->log_n = c->log_n;
    out->n = c->n;
    out->num_q = c->nq;
    out->num_p = c->np;
    out->dnum = c->dnum;
    out->alpha = c->alpha;
    out->level = level;
    out->beta = c->beta(level);
    for (u32 j = 0; j < out->beta && j < HKS_MAX_DIGITS; j++) {
        out->digit_lo[j] = c->digit_lo(j);
        out->digit_hi[j] = c->digit_hi(level, j);
    }
    out->device = c->device;
    return HKS_OK;
}

extern "C" hks_status hks_ctx_psi(const hks_ctx *c, uint32_t prime_idx, uint64_t *psi) {
    if (!c || !psi) HKS_FAIL(HKS_EINVAL, "ctx_psi: NULL argument");
    if (prime_idx >= c->primes.size()) HKS_FAIL(HKS_EINVAL, "ctx_psi: prime index %u out of range", prime_idx);
    *psi = c->psi[prime_idx];
    return HKS_OK;
}

void hks_func_smem(const void *fn, size_t smem) {
    static std::mutex mu;
    static std::set<std::pair<int, const void *>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert({dev, fn}).second) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int hks_num_sms() {
    // relaxed atomics: concurrent first calls from several host threads may both query the attribute,
    // and both store the same value
    static std::atomic<int> nsm[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = nsm[dev].load(std::memory_order_relaxed);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        nsm[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}
