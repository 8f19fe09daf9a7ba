// Probe 2: as tc05_probe.cu with 128-byte-swizzled K-major operands (K = 32
// tf32 per row = one swizzle atom; four K = 8 MMAs per tile, the descriptor
// start advanced 32 B per step) — does the layout change the per-MMA cost?
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// element (r, k) of an R x 32 tile, 128B swizzle: 8-row atoms of 1024 B
__host__ __device__ inline int swz_off(int r, int k) {
    const int chunk = (k >> 2) ^ (r & 7);
    return ((r >> 3) * 1024 + (r & 7) * 128 + chunk * 16) / 4 + (k & 3);
}
__device__ __forceinline__ uint64_t smem_desc_swz(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;               // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;     // SBO: next 8-row atom
    d |= (uint64_t)1 << 46;               // version
    d |= (uint64_t)2 << 61;               // SWIZZLE_128B
    return d;
}
__host__ __device__ inline uint32_t instr_desc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done) : "r"(su32(b)), "r"(phase) : "memory");
    } while (!done);
}

template <int N>
__global__ void __launch_bounds__(128)
probe_k(const float *A, const float *B, float *D, int reps, int mode, unsigned long long *cyc) {
    extern __shared__ __align__(1024) float dyn[];
    float *sA = dyn, *sB = dyn + 128 * 32;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 32; i += 128) sA[swz_off(i / 32, i % 32)] = A[i];
    for (int i = tid; i < N * 32; i += 128) sB[swz_off(i / 32, i % 32)] = B[i];
    int ncols = N < 32 ? 32 : N;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(&tmem_base)), "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base, idesc = instr_desc_tf32(128, N);
    if (tid == 0) {
        const unsigned long long t0 = clock64();
        for (int i = 0; i < reps; ++i)
#pragma unroll
            for (int s = 0; s < 4; ++s)
                mma_tf32(tbase, smem_desc_swz(su32(sA) + 32 * s), smem_desc_swz(su32(sB) + 32 * s),
                         idesc, (i > 0 || s > 0) ? 1u : 0u);
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                su32(&bar)));
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    } else {
        mbar_wait(&bar, 0);
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (mode == 0)
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + (uint32_t)c;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]),
                           "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            if (blockIdx.x == 0)
                for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
        }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                     "r"(ncols));
}

template <int N>
static void run(int sms) {
    std::vector<float> hA(128 * 32), hB(N * 32), hD(128 * N), ref(128 * N);
    srand(2);
    for (auto &v : hA) v = (float)(rand() % 17 - 8) / 8.0f;
    for (auto &v : hB) v = (float)(rand() % 17 - 8) / 8.0f;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < 32; ++k) s += (double)hA[m * 32 + k] * hB[n * 32 + k];
            ref[m * N + n] = (float)(2 * s);  // reps = 2
        }
    float *A, *B, *D;
    unsigned long long *cyc;
    cudaMalloc(&A, hA.size() * 4); cudaMalloc(&B, hB.size() * 4);
    cudaMalloc(&D, hD.size() * 4); cudaMalloc(&cyc, sms * 64);
    cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)(128 + N) * 32 * 4 + 1024;
    cudaFuncSetAttribute(probe_k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe_k<N><<<1, 128, smem>>>(A, B, D, 2, 0, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("N=%d error %s\n", N, cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(hD.data(), D, hD.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < 128 * N; ++i) maxerr = fmax(maxerr, fabs(hD[i] - ref[i]));
    const int reps = 1 << 14;
    for (int cps : {1, 2, 4}) {
        if (N * cps > 512) break;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        probe_k<N><<<sms * cps, 128, smem>>>(A, B, D, reps, 1, cyc);
        cudaEventRecord(e0);
        probe_k<N><<<sms * cps, 128, smem>>>(A, B, D, reps, 1, cyc);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c0; cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
        const double flops = 2.0 * 128 * N * 32 * (double)reps * sms * cps;
        printf("swz128 N=%3d CTAs/SM=%d: check %.3g; %.1f clk per K=8 MMA per issuer; %.1f TFLOP/s\n",
               N, cps, maxerr, (double)c0 / (4.0 * reps), flops / (ms * 1e-3) / 1e12);
    }
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<8>(sms); run<16>(sms); run<32>(sms); run<64>(sms); run<128>(sms); run<256>(sms);
    return 0;
}
