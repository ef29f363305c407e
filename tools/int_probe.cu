// tools/int_probe.cu -- step-0 calibration: integer-pipe throughput on B200.
//
// Measures, register-resident with 8 independent chains per thread and a full grid (148 SMs x
// 8 x 256 threads): IMAD (mad.lo.u32), IMAD.WIDE.U32 (mad.wide.u32), IMAD.HI (mad.hi.u32),
// IADD3 (add.u32), LOP3 (xor), FFMA, DFMA, and two 64-bit modular butterflies (exact Shoup and the
// approximate-quotient Shoup).  Prints one JSON object: lanes per clock per SM and ops/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_probe int_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2507_04775_b200/csrc/modarith.cuh"


#define ITERS 4096
#define CH 8

template <int OP>
__global__ void __launch_bounds__(256) k_probe(u32 *out, u32 seed) {
    u32 x[CH];
    u64 w[CH];
    float f[CH];
    double d[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) {
        x[c] = seed * (threadIdx.x + 1) + c;
        w[c] = ((u64)x[c] << 20) | c;
        f[c] = (float)x[c];
        d[c] = (double)x[c];
    }
    const u32 a = seed | 1, b = seed ^ 0x9e3779b9u;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            if (OP == 1) asm volatile("{.reg .u32 lo; cvt.u32.u64 lo, %0; mad.wide.u32 %0, lo, %1, %0;}" : "+l"(w[c]) : "r"(a));
            if (OP == 2) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            if (OP == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
            if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(x[(c + 1) % CH]), "r"(x[(c + 3) % CH]));
            if (OP == 5) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(1.0001f), "f"(0.5f));
            if (OP == 6) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(1.0001), "d"(0.5));
        }
    }
    u32 r = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) r ^= x[c] ^ (u32)w[c] ^ (u32)(w[c] >> 32) ^ __float_as_uint(f[c]) ^ (u32)__double_as_longlong(d[c]);
    if (r == 0x12345678) out[0] = r;
}

// 64-bit modular butterflies, p < 2^60.

template <int VAR>
__global__ void __launch_bounds__(256) k_bfly(u64 *out, u64 p, u64 w, u64 wp) {
    u64 X[CH], Y[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) {
        X[c] = (p >> 3) * (c + 1) + threadIdx.x;
        Y[c] = (p >> 2) + c * 977 + blockIdx.x;
    }
    const u64 two_p = 2 * p, four_p = 4 * p;
    const NttMod M = make_nttmod(p);
    for (int it = 0; it < ITERS / 8; it++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            if (VAR == 0) {   // exact Shoup, Harvey lazy [0,4p)
                u64 x = csub(X[c], two_p);
                u64 q = __umul64hi(Y[c], wp);
                u64 t = Y[c] * w - q * p;
                X[c] = x + t;
                Y[c] = x - t + two_p;
            } else if (VAR == 2) {   // library butterfly (ct_lazy, PTX Shoup)
                ct_lazy(X[c], Y[c], w, wp, M);
            } else if (VAR == 3) {   // library inverse butterfly (gs_lazy)
                gs_lazy(X[c], Y[c], w, wp, M);
            } else {          // approximate quotient (3 partial products), values in [0,8p)
                u64 x = csub(X[c], four_p);
                u64 y = Y[c];
                u32 yl = (u32)y, yh = (u32)(y >> 32), wl = (u32)wp, wh = (u32)(wp >> 32);
                u64 mid = (u64)__umulhi(yh, wl) + __umulhi(yl, wh);
                u64 q = (u64)yh * wh + mid;
                u64 t = y * w - q * p;
                X[c] = x + t;
                Y[c] = x - t + four_p;
            }
        }
    }
    u64 r = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) r ^= X[c] ^ Y[c];
    if (r == 0x1234567812345678ull) out[0] = r;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    u32 *o32;
    u64 *o64;
    cudaMalloc(&o32, 64);
    cudaMalloc(&o64, 64);
    const int blocks = sms * 8, threads = 256;
    const double lanes = (double)blocks * threads;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[7] = {"imad_lo", "imad_wide", "imad_hi", "iadd", "lop_xor", "ffma", "dfma"};
    printf("{\"sms\": %d, \"clock_khz_attr\": %d", sms, clk_khz);
    auto run = [&](auto kern, const char *name, double ops_per_lane) {
        for (int w = 0; w < 2; w++) kern();
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; r++) kern();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = lanes * ops_per_lane * reps;
        double per_s = ops / (ms * 1e-3);
        printf(", \"%s\": {\"ops_per_s\": %.4e, \"per_clk_per_sm_at_1965MHz\": %.2f}", name, per_s,
               per_s / (sms * 1.965e9));
    };
    run([&] { k_probe<0><<<blocks, threads>>>(o32, 7); }, names[0], (double)ITERS * CH);
    run([&] { k_probe<1><<<blocks, threads>>>(o32, 7); }, names[1], (double)ITERS * CH);
    run([&] { k_probe<2><<<blocks, threads>>>(o32, 7); }, names[2], (double)ITERS * CH);
    run([&] { k_probe<3><<<blocks, threads>>>(o32, 7); }, names[3], (double)ITERS * CH);
    run([&] { k_probe<4><<<blocks, threads>>>(o32, 7); }, names[4], (double)ITERS * CH);
    run([&] { k_probe<5><<<blocks, threads>>>(o32, 7); }, names[5], (double)ITERS * CH);
    run([&] { k_probe<6><<<blocks, threads>>>(o32, 7); }, names[6], (double)ITERS * CH);
    const u64 p = 0xffffffffffc0001ull, w = 0x123456789abcdefull % p;
    const u64 wp = (u64)(((unsigned __int128)w << 64) / p);
    run([&] { k_bfly<0><<<blocks, threads>>>(o64, p, w, wp); }, "bfly_shoup_exact", (double)ITERS / 8 * CH);
    run([&] { k_bfly<1><<<blocks, threads>>>(o64, p, w, wp); }, "bfly_shoup_approx", (double)ITERS / 8 * CH);
    run([&] { k_bfly<2><<<blocks, threads>>>(o64, p, w, wp); }, "bfly_ct_lazy_ptx", (double)ITERS / 8 * CH);
    run([&] { k_bfly<3><<<blocks, threads>>>(o64, p, w, wp); }, "bfly_gs_lazy_ptx", (double)ITERS / 8 * CH);
    printf("}\n");
    return 0;
}
