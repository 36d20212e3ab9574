// INT8 tensor-core (tcgen05.mma kind::i8, UTCIMMA) throughput on the B200:
// the ceiling a tensor-core NTT would work against.  One CTA
// per SM issues back-to-back M=128 x N=256 x K=32 s8 x s8 -> s32 MMAs from
// shared memory into a TMEM accumulator (operands are zeros: only the issue
// rate is measured).  Prints JSON lines with MACs per clock per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 imma_bench.cu -o imma_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 128, N = 256, K = 32;

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;            // descriptor version (sm100)
    return d;                          // base offset 0, SWIZZLE_NONE
}

__global__ void __launch_bounds__(128, 1) imma_kernel(int iters, long long *cycles) {
    __shared__ __align__(1024) int8_t A[M * K];
    __shared__ __align__(1024) int8_t B[N * K];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t taddr;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < M * K; i += blockDim.x) A[i] = 0;
    for (int i = tid; i < N * K; i += blockDim.x) B[i] = 0;
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&taddr);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(dst) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        // K-major, no swizzle: 8-row x 16-byte core matrices; two along K (LBO = 128 B),
        // 8-row groups SBO = 256 B apart
        const uint64_t da = smem_desc((uint32_t)__cvta_generic_to_shared(A), 128, 256);
        const uint64_t db = smem_desc((uint32_t)__cvta_generic_to_shared(B), 128, 256);
        uint32_t idesc = 0;
        idesc |= 2u << 4;                  // C format: S32
        idesc |= 1u << 7;                  // A format: signed 8 bit
        idesc |= 1u << 10;                 // B format: signed 8 bit
        idesc |= (uint32_t)(N >> 3) << 17; // N
        idesc |= (uint32_t)(M >> 4) << 24; // M
        const long long t0 = clock64();
        for (int i = 0; i < iters; i++) {
            const uint32_t acc = i > 0;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(taddr), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb)
                     : "memory");
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done)
                         : "r"(mb)
                         : "memory");
        }
        const long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(taddr) : "memory");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *d_cyc = nullptr;
    cudaMalloc(&d_cyc, sizeof(long long) * sms);
    for (int iters : {1000, 20000}) {
        imma_kernel<<<sms, 128>>>(10, d_cyc);   // warm-up
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        imma_kernel<<<sms, 128>>>(iters, d_cyc);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[1024];
        cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < sms; i++) cyc += (double)h[i];
        cyc /= sms;
        const double macs = (double)iters * M * N * K;
        printf("{\"op\": \"tcgen05.mma kind::i8 M128 N256 K32\", \"iters\": %d, \"mac_per_clk_per_sm\": %.1f, "
               "\"tera_mac_per_s\": %.1f, \"event_ms\": %.3f, \"err\": \"%s\"}\n",
               iters, macs / cyc, macs * sms / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(err));
    }
    return 0;
}
