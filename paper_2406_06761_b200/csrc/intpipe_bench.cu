// Integer-pipe and TMEM microbenchmarks: measure, on
// the B200 itself, the per-SM per-clock throughput of the instructions the
// hot path is made of, so the roofline denominator of the fused kernel is a
// measured number rather than a datasheet guess.
//
//   imad      x = x * a + b            (IMAD, FMA-heavy pipe)
//   imad_hi   x = umulhi(x, a)         (IMAD.HI)
//   iadd3     x0 = x0 + x1 + x2 ...    (IADD3, ALU pipe; rotating operands, not foldable)
//   shoup     x = shoup_mul(x, w, wp)  (3 IMAD-pipe instructions: one modmul)
//   gs_bfly   (X, Y) <- Harvey GS butterfly (3 IMAD + 3 ALU)
//   hi+lo     independent IMAD.HI and IMAD, 1:1 (the Shoup mix without its dependency)
//   imad+iadd independent IMAD and IADD3, 1:1 (FMA-heavy and ALU pipes together)
//   imad_wide IMAD.WIDE.U32 (+ LOP3 folding the two halves)
//   tmem_ld   tcgen05.ld.32x32b.x16 from tensor memory (bytes per clock per SM)
//
// Every thread runs CHAINS independent dependency chains; exactly one wave of
// CTAs is launched (occupancy-derived), and every CTA records clock64() and
// %globaltimer around its loop, so the report gives both the per-SM-clock rate
// and the SM clock the GPU actually ran at (cycles / ns).
// Output: one JSON line per op.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ntt_device.cuh"

using namespace wally;

static uint32_t g_iters = 1 << 15;  // argv[1] overrides (short runs under ncu)
constexpr int CHAINS = 8;
constexpr int REP = 2;  // chain steps per loop iteration

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int OP>
__global__ void __launch_bounds__(1024) bench_kernel(uint32_t iters, uint32_t a, uint32_t b, uint32_t q,
                                                     uint32_t *sink, unsigned long long *rec) {
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
    const long long t0 = clock64();
    const uint64_t g0 = gtimer();
    for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
        for (int rep = 0; rep < REP; rep++)
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            // volatile asm: one instruction per chain step
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            if (OP == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
            if (OP == 2) x[c] = x[c] + y[c] + x[(c + 1) % CHAINS];
            if (OP == 3) x[c] = shoup_mul(x[c], a, wp, q);
            if (OP == 4) gs_bfly(x[c], y[c], a, wp, q, 2 * q);
            if (OP == 5) {  // independent IMAD.HI + IMAD (1:1)
                asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(a), "r"(b));
            }
            if (OP == 6) {  // independent IMAD + IADD3 (1:1): FMA-heavy and ALU pipes together
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
                y[c] = y[c] + x[(c + 3) % CHAINS] + y[(c + 1) % CHAINS];
            }
            if (OP == 7) {  // IMAD.WIDE.U32 (+ LOP3 folding the halves)
                const uint64_t w64 = (uint64_t)x[c] * a;
                x[c] = (uint32_t)w64 ^ (uint32_t)(w64 >> 32);
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    const uint64_t g1 = gtimer();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s ^= x[c] ^ y[c];
    if (s == 0x12345678u) sink[0] = s;
    if (threadIdx.x == 0) {
        rec[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
        rec[2 * blockIdx.x + 1] = (unsigned long long)(g1 - g0);
    }
}

// FP64 pipe (round 2: could a second, double-precision modular multiplier
// run beside the IMAD pipe?):
//   10 dfma      x = fma(x, a, b)                    (DFMA)
//   11 cvt       x = (double)(uint32)x round trip     (F2I.F64 + I2F.F64)
//   12 fp64_mod  exact x * w mod q in doubles: h = x w, l = fma(x, w, -h),
//                t = rint(h / q), r = fma(-t, q, h) + l   (6 FP64 ops)
//   13 mixed     one Shoup modmul (IMAD pipe) and one fp64_mod per step, independent
template <int OP>
__global__ void __launch_bounds__(1024) fp64_kernel(uint32_t iters, uint32_t a, uint32_t b, uint32_t q,
                                                    uint32_t *sink, unsigned long long *rec) {
    double x[CHAINS];
    uint32_t u[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
        u[c] = (threadIdx.x * 7919u + c * 104729u + blockIdx.x) % q;
        x[c] = (double)u[c];
    }
    const double ad = (double)a, bd = (double)b, qd = (double)q, qinv = 1.0 / (double)q;
    const uint32_t wp = (uint32_t)(((uint64_t)a << 32) / q);
    __syncthreads();
    const long long t0 = clock64();
    const uint64_t g0 = gtimer();
    for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
        for (int rep = 0; rep < REP; rep++)
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            if (OP == 10) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(ad), "d"(bd));
            if (OP == 11) {
                uint32_t t;
                asm volatile("cvt.rzi.u32.f64 %0, %1;" : "=r"(t) : "d"(x[c]));
                asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(x[c]) : "r"(t + 1u));
            }
            if (OP == 12 || OP == 13) {
                const double h = x[c] * ad;
                const double l = fma(x[c], ad, -h);
                const double t = rint(h * qinv);
                x[c] = fma(-t, qd, h) + l;
            }
            if (OP == 13) u[c] = shoup_mul(u[c], a, wp, q);
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    const uint64_t g1 = gtimer();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s ^= (uint32_t)(int64_t)x[c] ^ u[c];
    if (s == 0x12345678u) sink[0] = s;
    if (threadIdx.x == 0) {
        rec[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
        rec[2 * blockIdx.x + 1] = (unsigned long long)(g1 - g0);
    }
}

// TMEM read bandwidth: 512 threads (16 warps), one CTA per SM, 512 columns
// allocated; warp w reads its lane quadrant (w % 4), columns (w / 4) * 128 + ...
__global__ void __launch_bounds__(512, 1) tmem_kernel(uint32_t iters, uint32_t *sink, unsigned long long *rec) {
    __shared__ uint32_t s_taddr;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_taddr);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = s_taddr + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)((warp / 4) * 128);
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    const uint64_t g0 = gtimer();
    for (uint32_t i = 0; i < iters; i++) {
        uint32_t r[16];
        const uint32_t addr = base + (i % 8) * 16;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 16; k++) acc += r[k];
    }
    __syncthreads();
    const long long t1 = clock64();
    const uint64_t g1 = gtimer();
    if (acc == 0x12345678u) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_taddr));
    if (threadIdx.x == 0) {
        rec[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
        rec[2 * blockIdx.x + 1] = (unsigned long long)(g1 - g0);
    }
}

// Rates from the kernel's elapsed time (CUDA events around the launch) and
// the SM clock: ops / (SMs x elapsed seconds x clock).  The clock is the
// ratio of a block's clock64 window to its globaltimer window (both taken
// inside the same block, so the ratio is valid even though the windows of
// co-resident blocks overlap -- dividing ops by those windows, as round 1
// did, double-counts co-resident blocks and overstates the rate).
static void report(const char *name, double ops_per_block, int blocks, int blocks_per_sm, int num_sms, float ms,
                   const unsigned long long *h, const char *unit) {
    double cyc = 0, ns = 0;
    for (int i = 0; i < blocks; i++) {
        cyc += (double)h[2 * i];
        ns += (double)h[2 * i + 1];
    }
    cyc /= blocks;
    ns /= blocks;
    const double clk_hz = cyc / ns * 1e9;
    const double total = ops_per_block * blocks;
    const double per_clk = total / num_sms / (ms * 1e-3 * clk_hz);
    printf("{\"op\": \"%s\", \"%s_per_clk_per_sm\": %.2f, \"tera_per_s\": %.3f, \"blocks_per_sm\": %d, "
           "\"sm_clock_mhz\": %.0f, \"event_ms\": %.3f, \"basis\": \"kernel elapsed (CUDA events) x SM clock\", "
           "\"err\": \"%s\"}\n",
           name, unit, per_clk, total / (ms * 1e-3) / 1e12, blocks_per_sm, clk_hz / 1e6, ms,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
}

template <int OP>
static auto kernel_of() {
    if constexpr (OP >= 10) return fp64_kernel<OP>;
    else return bench_kernel<OP>;
}

template <int OP>
static void run(const char *name, int num_sms, int ops_per_step = 1) {
    const int threads = 1024;
    int bps = 0;
    auto kern = kernel_of<OP>();
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, threads, 0);
    if (bps < 1) bps = 1;
    const int blocks = num_sms * bps;
    const uint32_t iters = g_iters;
    uint32_t *sink;
    unsigned long long *rec;
    cudaMalloc(&sink, 4);
    cudaMalloc(&rec, sizeof(unsigned long long) * 2 * blocks);
    const uint32_t q = 1073651713u, a = 123456789u, b = 987654321u;
    kern<<<blocks, threads>>>(1024, a, b, q, sink, rec);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(iters, a, b, q, sink, rec);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long *h = new unsigned long long[2 * blocks];
    cudaMemcpy(h, rec, sizeof(unsigned long long) * 2 * blocks, cudaMemcpyDeviceToHost);
    report(name, (double)threads * iters * CHAINS * REP * ops_per_step, blocks, bps, num_sms, ms, h, "thread_ops");
    delete[] h;
    cudaFree(sink);
    cudaFree(rec);
}

static void run_tmem(int num_sms) {
    const int blocks = num_sms;
    const uint32_t iters = 1 << 16;
    uint32_t *sink;
    unsigned long long *rec;
    cudaMalloc(&sink, 4);
    cudaMalloc(&rec, sizeof(unsigned long long) * 2 * blocks);
    tmem_kernel<<<blocks, 512>>>(256, sink, rec);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tmem_kernel<<<blocks, 512>>>(iters, sink, rec);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long *h = new unsigned long long[2 * blocks];
    cudaMemcpy(h, rec, sizeof(unsigned long long) * 2 * blocks, cudaMemcpyDeviceToHost);
    report("tmem_ld_32x32b_x16", 512.0 * iters * 16 * 4, blocks, 1, num_sms, ms, h, "bytes");
    delete[] h;
    cudaFree(sink);
    cudaFree(rec);
}

int main(int argc, char **argv) {
    if (argc > 1) g_iters = (uint32_t)atoi(argv[1]);
    int num_sms = 0;
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("imad", num_sms);
    run<1>("imad_hi", num_sms);
    run<2>("iadd3", num_sms);
    run<3>("shoup_modmul", num_sms);
    run<4>("gs_butterfly", num_sms);
    run<5>("imad_hi_plus_imad_1to1", num_sms, 2);
    run<6>("imad_plus_iadd3_1to1", num_sms, 2);
    run<7>("imad_wide_plus_lop3", num_sms, 1);
    run<10>("dfma", num_sms);
    run<11>("cvt_f64_u32_round_trip", num_sms);
    run<12>("fp64_modmul", num_sms);
    run<13>("shoup_plus_fp64_modmul_1to1", num_sms, 2);
    run_tmem(num_sms);
    return 0;
}
