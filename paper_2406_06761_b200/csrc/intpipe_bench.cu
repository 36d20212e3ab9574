// Integer-pipe microbenchmark: measures, on the
// B200 itself, the per-SM per-clock throughput of the instructions the hot
// path is made of, so the roofline denominator of the fused kernel is a
// measured number rather than a datasheet guess.
//
//   imad      x = x * a + b            (IMAD, FMA-heavy pipe)
//   imad_hi   x = umulhi(x, a)         (IMAD.HI)
//   iadd      x = x + b                (IADD3, ALU pipe)
//   shoup     x = shoup_mul(x, w, wp)  (3 IMAD-pipe instructions: one modmul)
//   gs_bfly   (X, Y) <- Harvey GS butterfly (3 IMAD + 3 ALU)
//
// Every thread runs CHAINS independent dependency chains, one resident wave
// fills all SMs (2 x 1024 threads per SM), and cycles are read with clock64()
// inside each block so the result is per SM-clock, independent of DVFS.
// Output: one JSON line per op: ops/clk/SM (thread-ops) and the wall rate.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "ntt_device.cuh"

using namespace wally;

constexpr int CHAINS = 8;

template <int OP>
__global__ void __launch_bounds__(1024) bench_kernel(uint32_t iters, uint32_t a, uint32_t b, uint32_t q,
                                                     uint32_t *sink, unsigned long long *cycles) {
    uint32_t x[CHAINS], y[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
        x[c] = threadIdx.x * 7919u + c * 104729u + blockIdx.x;
        y[c] = x[c] ^ 0x5bd1e995u;
        x[c] %= q;
        y[c] %= q;
    }
    const uint32_t wp = (uint32_t)(((uint64_t)a << 32) / q);
    __syncthreads();
    long long t0 = clock64();
    for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            // volatile asm: one instruction per chain step, never folded across iterations
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            if (OP == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
            if (OP == 2) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(b));
            if (OP == 3) x[c] = shoup_mul(x[c], a, wp, q);
            if (OP == 4) gs_bfly(x[c], y[c], a, wp, q, 2 * q);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s ^= x[c] ^ y[c];
    if (s == 0x12345678u) sink[0] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int OP>
static void run(const char *name, int ops_per_iter_chain, int num_sms) {
    const int threads = 1024, blocks_per_sm = 2, blocks = num_sms * blocks_per_sm;
    const uint32_t iters = 1 << 16;
    uint32_t *sink;
    unsigned long long *cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, sizeof(unsigned long long) * blocks);
    const uint32_t q = 1073651713u, a = 123456789u, b = 987654321u;
    bench_kernel<OP><<<blocks, threads>>>(1024, a, b, q, sink, cyc);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench_kernel<OP><<<blocks, threads>>>(iters, a, b, q, sink, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long *h = new unsigned long long[blocks];
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost);
    double mean_cyc = 0;
    for (int i = 0; i < blocks; i++) mean_cyc += (double)h[i];
    mean_cyc /= blocks;
    const double ops_per_sm = (double)blocks_per_sm * threads * iters * CHAINS * ops_per_iter_chain;
    const double per_clk = ops_per_sm / mean_cyc;
    const double total = ops_per_sm * num_sms;
    printf("{\"op\": \"%s\", \"ops_per_clk_per_sm\": %.2f, \"tera_ops_per_s\": %.3f, \"mean_cycles\": %.0f, "
           "\"ms\": %.3f, \"implied_clock_mhz\": %.0f, \"err\": \"%s\"}\n",
           name, per_clk, total / (ms * 1e-3) / 1e12, mean_cyc, ms, mean_cyc / (ms * 1e3),
           cudaGetErrorString(cudaGetLastError()));
    delete[] h;
    cudaFree(sink);
    cudaFree(cyc);
}

int main() {
    int num_sms = 0;
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("imad", 1, num_sms);
    run<1>("imad_hi", 1, num_sms);
    run<2>("iadd3", 1, num_sms);
    run<3>("shoup_modmul", 1, num_sms);
    run<4>("gs_butterfly", 1, num_sms);
    return 0;
}
