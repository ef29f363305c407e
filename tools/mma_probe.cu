// tools/mma_probe.cu -- legacy warp-level integer MMA throughput on B200 (sm_100a).
//
// Question it answers: how many u8 x u8 -> s32 multiply-accumulates per clock per SM does
// `mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32` (SASS IMMA) sustain on sm_100a, register-resident,
// with CH independent accumulator fragments per warp and a full grid?  This bounds a base conversion
// whose 60x60-bit products are split into bytes (DESIGN.md §5 "BConv on the tensor pipe").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 2048

template <int CH>
__global__ void __launch_bounds__(256) k_mma(uint32_t *out, uint32_t seed) {
    uint32_t a0 = seed * (threadIdx.x + 1), a1 = a0 ^ 0x55, a2 = a0 + 7, a3 = a0 * 3;
    uint32_t b0 = seed ^ threadIdx.x, b1 = b0 + 11;
    int d[CH][4];
#pragma unroll
    for (int c = 0; c < CH; c++) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < CH; c++)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int r = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) r ^= d[c][0] ^ d[c][1] ^ d[c][2] ^ d[c][3];
    if (r == 0x12345678) out[0] = r;
}

template <int CH>
static void run(int sms, int clk_khz, int ctas_per_sm) {
    uint32_t *out;
    cudaMalloc(&out, 4);
    dim3 grid(sms * ctas_per_sm);
    k_mma<CH><<<grid, 256>>>(out, 3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) k_mma<CH><<<grid, 256>>>(out, 3 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = 5.0 * grid.x * 8.0 /*warps*/ * ITERS * CH * (16.0 * 8 * 32);
    const double rate = macs / (ms * 1e-3);
    printf("{\"op\": \"mma.sync.m16n8k32.u8\", \"chains\": %d, \"ctas_per_sm\": %d, \"int8_mac_per_s\": %.4e, "
           "\"mac_per_clk_per_sm\": %.1f}\n",
           CH, ctas_per_sm, rate, rate / (sms * (double)clk_khz * 1e3));
    cudaFree(out);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    run<1>(sms, clk, 4);
    run<2>(sms, clk, 4);
    run<4>(sms, clk, 4);
    run<8>(sms, clk, 4);
    run<4>(sms, clk, 8);
    return 0;
}
