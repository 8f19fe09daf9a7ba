// Probe 3: the tcgen05 conv's per-chunk MMA batch — 12 kind::tf32 MMAs
// (4 K-steps x hi*hi, hi*lo, lo*hi; 128B-swizzled operands, M = 128) into a
// fresh accumulator (two alternating), then a commit.  Per batch:
//   mode 0: commits never waited on (issue throughput);
//   mode 1: each batch's commit waited on before the next (batch latency);
//   mode 2: batch b waits for batch b-2's commit (the kernels' double buffer).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint32_t idesc(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(su32(b)), "r"(phase) : "memory");
    } while (!done);
}
template <int N>
__global__ void __launch_bounds__(128) batch_k(int reps, int mode, unsigned long long *cyc) {
    extern __shared__ __align__(1024) float dyn[];
    float *aH = dyn, *aL = aH + 128 * 32, *bH = aL + 128 * 32, *bL = bH + N * 32;
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (256 + 2 * N) * 32; i += 128) dyn[i] = (float)((i * 7) % 13 - 6) / 8.0f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(2 * N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase, id = idesc(N);
    if (tid == 0) {
        const unsigned long long t0 = clock64();
        for (int b = 0; b < reps; ++b) {
            if (mode == 2 && b >= 2) mbar_wait(&bar[b & 1], ((b - 2) >> 1) & 1);
            const uint32_t acc = tm + (uint32_t)((b & 1) * N);
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint64_t ah = desc(su32(aH) + 32 * s), al = desc(su32(aL) + 32 * s);
                const uint64_t bh = desc(su32(bH) + 32 * s), bl = desc(su32(bL) + 32 * s);
                mma(acc, ah, bh, id, s ? 1u : 0u);
                mma(acc, ah, bl, id, 1u);
                mma(acc, al, bh, id, 1u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[b & 1])));
            if (mode == 1) mbar_wait(&bar[b & 1], (b >> 1) & 1);
        }
        // drain: the last two batches
        for (int b = reps - 2; b < reps; ++b)
            if (b >= 0 && mode != 1) mbar_wait(&bar[b & 1], (b >> 1) & 1);
        cyc[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(2 * N));
}
template <int N>
static void run(int sms) {
    unsigned long long *cyc;
    cudaMalloc(&cyc, 8 * sms * 4);
    const size_t smem = (size_t)(256 + 2 * N) * 32 * 4 + 1024;
    cudaFuncSetAttribute(batch_k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 2048;
    for (int mode = 0; mode < 3; ++mode)
        for (int cps : {1, 2}) {
            batch_k<N><<<sms * cps, 128, smem>>>(reps, mode, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
            unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("N=%d mode=%d CTAs/SM=%d: %.0f clk per 12-MMA batch (%.1f per MMA)\n", N, mode, cps,
                   (double)c / reps, (double)c / reps / 12);
        }
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<32>(sms); run<64>(sms);
    return 0;
}
