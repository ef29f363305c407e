#include <stdlib.h>
// prof.cu -- launch counter and optional per-kernel CUDA-event timer (include/hks.h diagnostics).
#include <string.h>

#include <atomic>
#include <mutex>

#include "internal.h"

namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_on{0};
struct Rec {
    int cls;
    cudaEvent_t a, b;
    double bytes, muls;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
const char *g_names[K_NCLS] = {"ntt_fwd_cols", "ntt_fwd_rows", "ntt_fwd_rows_moddown", "ntt_inv_rows",
                               "ntt_inv_cols_scale", "bconv", "kip", "automorph", "ntt_rows_kip", "pt_wsum",
                               "add_ct", "ntt_inv_fused"};

cudaEvent_t get_event() {
    std::lock_guard<std::mutex> l(g_mu);
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

ProfScope::ProfScope(int c, cudaStream_t st) : cls(c), s(st) {
    if (g_on.load(std::memory_order_relaxed)) {
        a = get_event();
        cudaEventRecord(a, s);
    }
}

void ProfScope::done(double bytes, double muls) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!a) return;
    cudaEvent_t b = get_event();
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> l(g_mu);
    g_recs.push_back(Rec{cls, a, b, bytes, muls});
    a = nullptr;
}

extern "C" uint64_t hks_launch_count(void) { return g_launches.load(); }

bool prof_active() { return g_on.load(std::memory_order_relaxed) != 0; }

extern "C" hks_status hks_prof_enable(int on) {
    g_on.store(on ? 1 : 0);
    return HKS_OK;
}

extern "C" int hks_prof_read(hks_prof_entry *out, int max) {
    std::vector<Rec> recs;
    {
        std::lock_guard<std::mutex> l(g_mu);
        recs.swap(g_recs);
    }
    uint64_t n[K_NCLS] = {0};
    double ms[K_NCLS] = {0}, by[K_NCLS] = {0}, mu[K_NCLS] = {0};
    for (auto &r : recs) {
        float t = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&t, r.a, r.b);
        n[r.cls]++;
        ms[r.cls] += t;
        by[r.cls] += r.bytes;
        mu[r.cls] += r.muls;
    }
    {
        std::lock_guard<std::mutex> l(g_mu);
        for (auto &r : recs) {
            g_pool.push_back(r.a);
            g_pool.push_back(r.b);
        }
    }
    int k = 0;
    for (int c = 0; c < K_NCLS && k < max; c++) {
        if (!n[c]) continue;
        memset(&out[k], 0, sizeof(out[k]));
        strncpy(out[k].name, g_names[c], sizeof(out[k].name) - 1);
        out[k].launches = n[c];
        out[k].total_ms = ms[c];
        out[k].bytes = by[c];
        out[k].muls = mu[c];
        k++;
    }
    return k;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("HKS_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}
