// Probe: tcgen05.mma kind::tf32 (M = 128, K = 8 per instruction) from
// shared-memory operands (K-major, no swizzle) into TMEM — correctness of one
// tile against the CPU, then issue throughput for N = 8 .. 256 with several
// TMEM accumulators in flight.  The small-N rates are what an implicit-GEMM
// encoder convolution at 8-16 output channels would run at.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc05_probe tc05_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major, SWIZZLE_NONE: core matrices of 8 rows x 16 bytes (4 tf32),
// stored [row group (8 rows)][k core (4 elems)][8 rows][4 elems]
// element (r, k) of an R x 8 tile -> offset ((r/8)*2 + k/4)*32 + (r%8)*4 + k%4
__host__ __device__ inline int kmaj_off(int r, int k) {
    return ((r >> 3) * 2 + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ uint64_t smem_desc(const void *p, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((su32(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm100)
    // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
    return d;
}

__host__ __device__ inline uint32_t instr_desc_tf32(int M, int N) {
    uint32_t d = 0;
    d |= 1u << 4;                     // D = F32
    d |= 2u << 7;                     // A = TF32
    d |= 2u << 10;                    // B = TF32
    // a_major = b_major = K (0)
    d |= (uint32_t)(N >> 3) << 17;
    d |= (uint32_t)(M >> 4) << 24;
    return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(su32(b)), "r"(phase)
            : "memory");
    } while (!done);
}

// grid: one CTA per SM; 128 threads (4 warps).  mode 0: one MMA chain of
// `reps` K-steps over the same operands into accumulator 0 (for the check);
// mode 1: `reps` MMAs round-robin over `nacc` accumulators (throughput).
template <int N>
__global__ void __launch_bounds__(128)
probe_k(const float *A, const float *B, float *D, int reps, int mode, int nacc,
        unsigned long long *cycles) {
    __shared__ __align__(1024) float sA[128 * 8];
    __shared__ __align__(1024) float sB[N * 8];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 8; i += 128) {
        const int r = i / 8, k = i % 8;
        sA[kmaj_off(r, k)] = A[i];
    }
    for (int i = tid; i < N * 8; i += 128) {
        const int r = i / 8, k = i % 8;
        sB[kmaj_off(r, k)] = B[i];
    }
    // TMEM: enough columns for nacc accumulators of N fp32 columns (power of 2 >= 32)
    int ncols = 32;
    while (ncols < N * nacc) ncols <<= 1;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(&tmem_base)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;");  // smem writes visible to the tensor core
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base;
    const uint64_t da = smem_desc(sA, 128, 256), db = smem_desc(sB, 128, 256);
    const uint32_t idesc = instr_desc_tf32(128, N);
    unsigned long long t0 = 0, t1 = 0;
    if (tid == 0) {
        t0 = clock64();
        for (int i = 0; i < reps; ++i) {
            const uint32_t acc_col = mode == 0 ? 0u : (uint32_t)((i % nacc) * N);
            mma_tf32(tbase + acc_col, da, db, idesc, mode == 0 ? (i > 0) : (i >= nacc));
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                su32(&bar)));
    }
    mbar_wait(&bar, 0);
    if (tid == 0) {
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // accumulator 0 back: warp w reads TMEM lanes 32w..32w+31; 8 columns per load
    if (mode == 0) {
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + (uint32_t)c;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                  "=r"(v[6]), "=r"(v[7])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            if (blockIdx.x == 0)
                for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
        }
    }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                     "r"(ncols));
}

template <int N>
static void run(int sms) {
    std::vector<float> hA(128 * 8), hB(N * 8), hD(128 * N), ref(128 * N);
    srand(1);
    // values exactly representable in tf32 (10-bit mantissa): small integers / 8
    for (auto &v : hA) v = (float)(rand() % 17 - 8) / 8.0f;
    for (auto &v : hB) v = (float)(rand() % 17 - 8) / 8.0f;
    const int reps_check = 3;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < 8; ++k) s += (double)hA[m * 8 + k] * hB[n * 8 + k];
            ref[m * N + n] = (float)(s * reps_check);
        }
    float *A, *B, *D;
    unsigned long long *cyc;
    cudaMalloc(&A, hA.size() * 4);
    cudaMalloc(&B, hB.size() * 4);
    cudaMalloc(&D, hD.size() * 4);
    cudaMalloc(&cyc, sms * 8 * 8);
    cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(D, 0, hD.size() * 4);
    probe_k<N><<<1, 128>>>(A, B, D, reps_check, 0, 1, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%3d: error %s\n", N, cudaGetErrorString(e));
        exit(1);
    }
    cudaMemcpy(hD.data(), D, hD.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < 128 * N; ++i) maxerr = fmax(maxerr, fabs(hD[i] - ref[i]));
    // throughput: every SM issues reps MMAs over nacc accumulators
    const int reps = 1 << 16;
    for (int cps : {1, 2, 4})
    for (int nacc : {1, 2}) {
        if (N * nacc * cps > 512) break;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        probe_k<N><<<sms * cps, 128>>>(A, B, D, reps, 1, nacc, cyc);
        cudaEventRecord(e0);
        probe_k<N><<<sms * cps, 128>>>(A, B, D, reps, 1, nacc, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c0;
        cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
        const double flops = 2.0 * 128 * N * 8 * (double)reps * sms * cps;
        printf("N=%3d CTAs/SM=%d nacc=%d: check max|err| %.3g; %.1f clk per MMA per issuer; "
               "%.1f TFLOP/s (tf32)\n", N, cps, nacc, maxerr, (double)c0 / reps,
               flops / (ms * 1e-3) / 1e12);
    }
    cudaFree(A);
    cudaFree(B);
    cudaFree(D);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<8>(sms);
    run<16>(sms);
    run<32>(sms);
    run<64>(sms);
    run<128>(sms);
    run<256>(sms);
    return 0;
}
