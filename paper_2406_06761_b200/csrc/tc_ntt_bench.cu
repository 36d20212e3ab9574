// Tensor-core experiment (SURVEY.md §7 "Tensor-core note", B2-K6; north_star:
// tensor cores "only if a limb-split int8 formulation ... measurably beats the
// IMAD pipe", evidenced by ncu).  Standalone binary, not on the product path.
//
// The operation: one 64-point stage of a four-step NTT (N = 4096 = 64 x 64):
// for a batch of vectors x (64 residues mod q, q = the c3 limb q_0), the
// cyclic length-64 transform  y[k] = sum_j x[j] w^(j k) mod q,  w a primitive
// 64th root of unity mod q (the inverse transform is the same with w^-1;
// PAPER.md P:L1000 is the NTT this replaces).  Two kernels compute it:
//
//   imad_kernel  the integer-pipe reference: one vector per thread in
//                registers, six radix-2 Gentleman-Sande stages with Shoup
//                twiddle products (the fused kernel's arithmetic), 3 modmuls
//                per output.
//   tc_kernel    tcgen05.mma kind::i8 (UTCIMMA): x and W split into 4 unsigned
//                byte planes, W stacked in pairs [W_a; W_{a+1}] to fill M = 128,
//                2 x 4 x 2 MMAs (K = 32 each) per tile of 32 vectors into six
//                TMEM accumulator regions (the partial sums of equal byte
//                weight 2^(8 s)); epilogue per output: 6 TMEM words per half,
//                64-bit recombination, two Shoup reductions per half, halves
//                added through shared memory.
//
// Both are checked against a host computation on every output.  Printed:
// one JSON line per kernel (ms, outputs/s, ns per 1,000 outputs) and, with
// --mma-only, the tensor kernel without its epilogue (its MMA + split floor).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo tc_ntt_bench.cu -o tc_ntt_bench
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr uint32_t Q = 1073651713u;   // the c3 limb q_0 (reading S5)
constexpr int VN = 64;                // transform length
constexpr int TV = 32;                // vectors per tensor-core tile (MMA N)

// ---------------------------------------------------------------------------
// host number theory
// ---------------------------------------------------------------------------
static uint64_t mulm(uint64_t a, uint64_t b) { return (unsigned __int128)a * b % Q; }
static uint64_t powm(uint64_t b, uint64_t e) {
    uint64_t r = 1;
    for (b %= Q; e; e >>= 1, b = mulm(b, b))
        if (e & 1) r = mulm(r, b);
    return r;
}
static uint32_t root64() {
    for (uint64_t x = 2;; x++) {
        uint64_t w = powm(x, (Q - 1) / 64);
        if (powm(w, 32) == Q - 1) return (uint32_t)w;
    }
}
static uint32_t shoup(uint32_t w) { return (uint32_t)(((uint64_t)w << 32) / Q); }

// ---------------------------------------------------------------------------
// device arithmetic (as ntt_device.cuh)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t csub(uint32_t x, uint32_t m) { return min(x, x - m); }
__device__ __forceinline__ uint32_t shoup_mul(uint32_t x, uint32_t w, uint32_t wp) {
    return x * w - __umulhi(x, wp) * Q;
}

// ---------------------------------------------------------------------------
// IMAD reference: thread = vector; GS (decimation in frequency) with natural
// input, bit-reversed output written back in natural order
// ---------------------------------------------------------------------------
__constant__ uint2 c_tw[VN];   // stage s, butterfly offset o: w^(o * 2^s) for o < 32 >> s  (index (64 >> (s+1)) + o)

__global__ void __launch_bounds__(128) imad_kernel(const uint32_t *__restrict__ x, uint32_t *__restrict__ y,
                                                   uint32_t nvec, int reps) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nvec) return;
    uint32_t a[VN];
    const uint4 *src = reinterpret_cast<const uint4 *>(x + (size_t)v * VN);
#pragma unroll
    for (int i = 0; i < VN / 4; i++) {
        const uint4 t = __ldg(src + i);
        a[4 * i] = t.x; a[4 * i + 1] = t.y; a[4 * i + 2] = t.z; a[4 * i + 3] = t.w;
    }
    // DIF: stage with half-length h = 32, 16, ..., 1: (X, Y) -> (X + Y, (X - Y) w^(o * 64 / (2h))).
    // `reps` applications back to back in registers (the output, in bit-reversed order and canonical,
    // is the next application's input: a compute-bound measure of the same arithmetic)
#pragma unroll 1
    for (int rep = 0; rep < reps; rep++) {
    if (rep) {
        uint32_t t[VN];
#pragma unroll
        for (int k = 0; k < VN; k++) t[k] = csub(csub(a[__brev(k) >> 26], 2 * Q), Q);
#pragma unroll
        for (int k = 0; k < VN; k++) a[k] = t[k];
    }
#pragma unroll
    for (int s = 0; s < 6; s++) {
        const int h = 32 >> s;
#pragma unroll
        for (int b = 0; b < VN; b += 2 * h)
#pragma unroll
            for (int o = 0; o < h; o++) {
                const uint2 w = c_tw[h + o];
                const uint32_t X = a[b + o], Y = a[b + o + h];
                a[b + o] = csub(X + Y, 2 * Q);
                a[b + o + h] = shoup_mul(X - Y + 2 * Q, w.x, w.y);
            }
    }
    }
    uint32_t *dst = y + (size_t)v * VN;
#pragma unroll
    for (int k = 0; k < VN; k++) {
        const int r = __brev(k) >> 26;          // position of output k after DIF
        dst[k] = csub(csub(a[r], 2 * Q), Q);
    }
}

// ---------------------------------------------------------------------------
// tensor-core version
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;            // descriptor version (sm100)
    return d;                          // base offset 0, SWIZZLE_NONE
}
// K-major, no swizzle, K = 64 bytes per row: element (row r, k) at
// (r / 8) * 512 + (k / 16) * 128 + (r % 8) * 16 + k % 16   (LBO 128 along K, SBO 512 along rows)
__host__ __device__ __forceinline__ uint32_t kmaj(uint32_t r, uint32_t k) {
    return (r >> 3) * 512 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

constexpr int TC_THREADS = 128;
constexpr int NREG = 6;                         // accumulator regions (byte weights of the top half)
constexpr int TMEM_COLS = 256;                  // >= NREG * TV, power of two

struct TcSmem {
    uint8_t A[2][128 * VN];                     // [W_0; W_1], [W_2; W_3]   (8 KB each)
    uint8_t B[4][TV * VN];                      // byte planes of the x tile (2 KB each)
    uint32_t bot[VN][TV + 1];                   // bottom-half partial results
    uint64_t mbar;
    uint32_t taddr;
};

__global__ void __launch_bounds__(TC_THREADS, 1) tc_kernel(const uint8_t *__restrict__ wplanes, const uint32_t *__restrict__ x,
                                                           uint32_t *__restrict__ y, uint32_t ntiles, int mma_only, int reps,
                                                           uint32_t c32, uint32_t c32p, uint32_t one_p, uint32_t c256p) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    TcSmem &sm = *reinterpret_cast<TcSmem *>(smraw);
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < 2 * 128 * VN / 16; i += TC_THREADS)
        reinterpret_cast<uint4 *>(sm.A)[i] = __ldg(reinterpret_cast<const uint4 *>(wplanes) + i);
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm.taddr);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&sm.mbar);
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = sm.taddr;
    // instruction descriptor: D = S32, A = B = U8, both K-major, N = TV, M = 128
    const uint32_t idesc = (2u << 4) | ((uint32_t)(TV >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint32_t phase = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // split the tile's TV x 64 residues into four byte planes (B operands: row = vector, K = element)
        const uint32_t *xt = x + (size_t)tile * TV * VN;
        for (int i = tid; i < TV * VN / 4; i += TC_THREADS) {
            const int v = i / (VN / 4), k4 = (i % (VN / 4)) * 4;
            const uint4 t = __ldg(reinterpret_cast<const uint4 *>(xt + (size_t)v * VN + k4));
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const uint32_t word = __byte_perm(__byte_perm(t.x >> (8 * b), t.y >> (8 * b), 0x0040),
                                                  __byte_perm(t.z >> (8 * b), t.w >> (8 * b), 0x0040), 0x5410);
                *reinterpret_cast<uint32_t *>(&sm.B[b][kmaj(v, k4)]) = word;
            }
        }
#pragma unroll 1
        for (int rep = 0; rep < reps; rep++) {
        const bool last = rep + 1 == reps;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // region r (columns r * TV ..) accumulates A_pair p x plane b with 2p + b = r
            bool first[NREG] = {true, true, true, true, true, true};
#pragma unroll
            for (int p = 0; p < 2; p++)
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int r = 2 * p + b;
                    const uint32_t d = tbase + (uint32_t)(r * TV);
#pragma unroll
                    for (int kh = 0; kh < 2; kh++) {   // K = 64 as two K = 32 MMAs (2 core matrices along K each)
                        const uint64_t da = smem_desc((uint32_t)__cvta_generic_to_shared(sm.A[p]) + kh * 256, 128, 512);
                        const uint64_t db = smem_desc((uint32_t)__cvta_generic_to_shared(sm.B[b]) + kh * 256, 128, 512);
                        const uint32_t acc = first[r] ? 0u : 1u;
                        first[r] = false;
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
                    }
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb)
                         : "memory");
        }
        // wait for the MMAs (also frees the B planes for the next tile)
        {
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(done)
                             : "r"(mb), "r"(phase)
                             : "memory");
            phase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (!mma_only) {
            // epilogue: lane = row m of the stacked output (m < 64: top half W_{2p}, m >= 64: W_{2p+1})
            const int m = tid, k = m & 63;
            const bool top = m < 64;
            const uint32_t lane_base = tbase + ((uint32_t)(32 * warp) << 16);
#pragma unroll 1
            for (int n0 = 0; n0 < TV; n0 += 8) {
                uint32_t part[NREG][8];
#pragma unroll
                for (int r = 0; r < NREG; r++)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(part[r][0]), "=r"(part[r][1]), "=r"(part[r][2]), "=r"(part[r][3]),
                                   "=r"(part[r][4]), "=r"(part[r][5]), "=r"(part[r][6]), "=r"(part[r][7])
                                 : "r"(lane_base + (uint32_t)(r * TV + n0)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                uint32_t outv[8];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    // value = sum_r 2^(8 r) part[r] < 2^64 (the bottom half carries one more factor 2^8)
                    uint64_t v = 0;
#pragma unroll
                    for (int r = 0; r < NREG; r++) v += (uint64_t)part[r][j] << (8 * r);
                    const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
                    uint32_t res = shoup_mul(lo, 1u, one_p) + shoup_mul(hi, c32, c32p);   // < 4q
                    res = csub(csub(res, 2 * Q), Q);
                    if (top) outv[j] = res;
                    else sm.bot[k][n0 + j] = csub(shoup_mul(res, 256u, c256p), Q);
                }
                __syncthreads();
                if (top) {
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        const uint32_t r = csub(outv[j] + sm.bot[k][n0 + j], Q);
                        if (last) {
                            y[((size_t)tile * TV + n0 + j) * VN + k] = r;
                        } else {   // the next application's input: byte planes of the output, in place
#pragma unroll
                            for (int b = 0; b < 4; b++) sm.B[b][kmaj(n0 + j, k)] = (uint8_t)(r >> (8 * b));
                        }
                    }
                }
                __syncthreads();
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TMEM_COLS) : "memory");
}

int main(int argc, char **argv) {
    bool mma_only_too = false;
    int reps = 1;
    for (int i = 1; i < argc; i++) {
        if (!strcmp(argv[i], "--mma-only")) mma_only_too = true;
        if (!strcmp(argv[i], "--reps") && i + 1 < argc) reps = atoi(argv[++i]);
    }
    const uint32_t nvec = 1u << 20;              // 2^20 vectors x 64 residues = 256 MB in, 256 MB out
    const uint32_t ntiles = nvec / TV;
    const uint32_t w = root64();
    // host inputs
    std::vector<uint32_t> hx((size_t)nvec * VN);
    uint64_t st = 88172645463325252ull;
    for (auto &v : hx) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        v = (uint32_t)(st % Q);
    }
    // DFT matrix W[k][j] = w^(j k) and its byte planes, stacked: A_p rows 0..63 = plane 2p, 64..127 = plane 2p+1
    std::vector<uint8_t> hA(2 * 128 * VN);
    for (int k = 0; k < VN; k++)
        for (int j = 0; j < VN; j++) {
            const uint32_t Wkj = (uint32_t)powm(w, (uint64_t)j * k);
            for (int a = 0; a < 4; a++) {
                const int p = a / 2, row = (a % 2) * 64 + k;
                hA[(size_t)p * 128 * VN + kmaj(row, j)] = (uint8_t)(Wkj >> (8 * a));
            }
        }
    uint2 htw[VN] = {};
    for (int h = 1; h <= 32; h <<= 1)
        for (int o = 0; o < h; o++) {
            const uint32_t t = (uint32_t)powm(w, (uint64_t)o * (32 / h));
            htw[h + o] = make_uint2(t, shoup(t));
        }
    CK(cudaMemcpyToSymbol(c_tw, htw, sizeof htw));
    uint32_t *dx, *dy1, *dy2;
    uint8_t *dA;
    CK(cudaMalloc(&dx, hx.size() * 4));
    CK(cudaMalloc(&dy1, hx.size() * 4));
    CK(cudaMalloc(&dy2, hx.size() * 4));
    CK(cudaMalloc(&dA, hA.size()));
    CK(cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t tsm = sizeof(TcSmem);
    CK(cudaFuncSetAttribute(tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tc_kernel, TC_THREADS, tsm));
    const uint32_t c32 = (uint32_t)((1ull << 32) % Q);
    const int ctas = 2;     // TMEM: 256 columns per CTA, 512 per SM (shared memory allows more: occupancy API says %d)
    (void)occ;
    auto run_imad = [&]() { imad_kernel<<<(nvec + 127) / 128, 128>>>(dx, dy1, nvec, reps); };
    auto run_tc = [&](int mma_only) {
        tc_kernel<<<sms * ctas, TC_THREADS, tsm>>>(dA, dx, dy2, ntiles, mma_only, reps, c32, shoup(c32),
                                                   (uint32_t)((1ull << 32) / Q), shoup(256));
    };
    auto timeit = [&](auto fn) {
        for (int i = 0; i < 3; i++) fn();
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int reps = 20;
        cudaEventRecord(e0);
        for (int i = 0; i < reps; i++) fn();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        CK(cudaGetLastError());
        return ms / reps;
    };
    const float t_imad = timeit(run_imad);
    const float t_tc = timeit([&] { run_tc(0); });
    // check every output of both against the host definition
    std::vector<uint32_t> y1(hx.size()), y2(hx.size());
    CK(cudaMemcpy(y1.data(), dy1, hx.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y2.data(), dy2, hx.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> Wm(VN * VN);
    for (int k = 0; k < VN; k++)
        for (int j = 0; j < VN; j++) Wm[k * VN + j] = (uint32_t)powm(w, (uint64_t)j * k);
    size_t bad1 = 0, bad2 = 0;
    for (uint32_t v = 0; v < nvec; v += (v < 4096 ? 1 : 97)) {
        uint32_t cur[VN], nxt[VN];
        for (int j = 0; j < VN; j++) cur[j] = hx[(size_t)v * VN + j];
        for (int r = 0; r < reps; r++) {
            for (int k = 0; k < VN; k++) {
                unsigned __int128 s = 0;
                for (int j = 0; j < VN; j++) s += (unsigned __int128)Wm[k * VN + j] * cur[j];
                nxt[k] = (uint32_t)(s % Q);
            }
            memcpy(cur, nxt, sizeof cur);
        }
        for (int k = 0; k < VN; k++) {
            bad1 += y1[(size_t)v * VN + k] != cur[k];
            bad2 += y2[(size_t)v * VN + k] != cur[k];
        }
    }
    const double outs = (double)nvec * VN;
    printf("{\"kernel\": \"imad_kernel (6 radix-2 Shoup stages, 3 modmul/output)\", \"reps\": %d, \"ms\": %.4f, "
           "\"outputs_per_s\": %.4g, \"mismatches\": %zu}\n", reps, t_imad, outs * reps / (t_imad * 1e-3), bad1);
    printf("{\"kernel\": \"tc_kernel (tcgen05.mma kind::i8, 4x4 byte planes, TMEM recombination + reduction)\", "
           "\"ms\": %.4f, \"outputs_per_s\": %.4g, \"mismatches\": %zu, \"ctas_per_sm\": %d, \"vs_imad\": %.3f}\n",
           t_tc, outs * reps / (t_tc * 1e-3), bad2, ctas, t_tc / t_imad);
    if (mma_only_too) {
        const float t_m = timeit([&] { run_tc(1); });
        printf("{\"kernel\": \"tc_kernel --mma-only (byte split once + reps x MMAs, no epilogue: the tensor floor)\", "
               "\"reps\": %d, \"ms\": %.4f, \"vs_imad\": %.3f}\n", reps, t_m, t_m / t_imad);
    }
    return (bad1 || bad2) ? 1 : 0;
}
