// Experiment: the encoder's 3x3x3 convolution (zero padded, ops.hpp:58-74) as
// an implicit GEMM on the 5th-generation tensor cores: D[voxel][oc] =
// sum_k A[voxel][k] B[oc][k], k = tap * ic + c, with fp32 accuracy from
// 3xTF32 (hi*hi + hi*lo + lo*hi).  One CTA = 128 consecutive output voxels
// (M = 128); per K chunk of 32 the 128 threads gather their voxel's 32
// values (im2col on the fly), split them into tf32 hi / lo and store them
// 128-byte swizzled K-major in shared memory; one thread issues the 12
// tcgen05.mma (4 K-steps x 3 products) into a TMEM accumulator of N = oc
// columns; the epilogue reads TMEM back (tcgen05.ld), adds the bias and
// writes the planar output.  dev experiment: compared with
// mdg_encoder_conv3_fwd in tcconv_bench.py.
#include <cuda_runtime.h>
#include <cstdint>

namespace {

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// element (r, k) of an R x 32 fp32 tile, 128B swizzle (8-row atoms of 1 KB)
__device__ __forceinline__ int swz(int r, int k) {
    return ((r >> 3) * 1024 + (r & 7) * 128 + (((k >> 2) ^ (r & 7)) << 4)) / 4 + (k & 3);
}
__device__ __forceinline__ uint64_t desc_swz(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) |
           ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint32_t idesc_tf32(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ float tf32r(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
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

// weights w {oc, ic, 3, 3, 3} -> B hi / lo {oc, Kp} (k = tap * ic + c, zero padded)
__global__ void prep_b(const float *w, int oc, int ic, int Kp, float *bhi, float *blo) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= oc * Kp) return;
    const int o = i / Kp, k = i % Kp;
    float v = 0.0f;
    if (k < 27 * ic) {
        const int tap = k / ic, c = k % ic;
        v = w[((int64_t)o * ic + c) * 27 + tap];
    }
    const float h = tf32r(v);
    bhi[i] = h;
    blo[i] = tf32r(v - h);
}

// A and B values of one K chunk for this thread, in registers (ic % 16 == 0)
template <int N>
struct ChunkRegs {
    static constexpr int BPT = (N * 32 + 255) / 256;
    float a[16], bh[BPT], bl[BPT];
};

template <int N>
__device__ __forceinline__ void load_chunk(ChunkRegs<N> &R, int j, int half, int tid, bool live,
                                           int x, int y, int z, int h, int w, int l, int64_t n,
                                           int ic, int K27, int Kp, const float *__restrict__ in,
                                           const float *__restrict__ bhi,
                                           const float *__restrict__ blo) {
#pragma unroll
    for (int u = 0; u < ChunkRegs<N>::BPT; ++u) {
        const int e = tid + 256 * u;
        if (e < N * 32) {
            const int r = e >> 5, kk = e & 31;
            R.bh[u] = __ldg(bhi + (int64_t)r * Kp + 32 * j + kk);
            R.bl[u] = __ldg(blo + (int64_t)r * Kp + 32 * j + kk);
        }
    }
    const int k = 32 * j + 16 * half;
    const int tap = k < K27 ? k / ic : 27;
    const int c0 = k - tap * ic;
    bool ok = false;
    int64_t off = 0;
    if (tap < 27 && live) {
        const int xx = x + tap % 3 - 1, yy = y + (tap / 3) % 3 - 1, zz = z + tap / 9 - 1;
        ok = xx >= 0 && xx < h && yy >= 0 && yy < w && zz >= 0 && zz < l;
        off = (int64_t)c0 * n + ((int64_t)zz * w + yy) * h + xx;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) R.a[q] = ok ? __ldg(in + off + (int64_t)q * n) : 0.0f;
}

template <int N>
__global__ void __launch_bounds__(256)
tcconv_k(const float *__restrict__ in, int ic, int h, int w, int l, const float *__restrict__ bhi,
         const float *__restrict__ blo, int Kp, const float *__restrict__ bias,
         float *__restrict__ out) {
    extern __shared__ __align__(1024) float sm_raw[];
    // the swizzle atoms must start on 1 KB boundaries of the shared window
    float *sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u) / 4;
    constexpr int STAGE = 2 * 128 * 32 + 2 * N * 32;  // floats per pipeline stage
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int row = tid & 127, half = tid >> 7;  // voxel row, K half of each chunk
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * 128 + row;
    const bool live = p < n;
    int x = 0, y = 0, z = 0;
    if (live) {
        const int t = (int)(p / h);
        x = (int)(p - (int64_t)t * h);
        z = t / w;
        y = t - z * w;
    }
    constexpr int NCOL = 2 * N < 32 ? 32 : 2 * N;  // two accumulators (ping-pong)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(&tmem_base)), "r"(NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base, id = idesc_tf32(N);
    const int nchunk = Kp / 32, K27 = 27 * ic;
    // software pipeline: chunk j+1's global loads are in flight while chunk
    // j is split, stored and handed to the tensor core
    ChunkRegs<N> R;
    load_chunk<N>(R, 0, half, tid, live, x, y, z, h, w, l, n, ic, K27, Kp, in, bhi, blo);
    // each chunk's 12 MMAs accumulate into a fresh TMEM accumulator (alternating
    // between two); the chunk sums are added in fp32 registers, RN, in chunk
    // order — the tensor core never accumulates across chunks.  Warps w and
    // w+4 read TMEM lanes 32(w%4).. for the column halves [0, N/2), [N/2, N).
    constexpr int NH = N / 2;
    float acc[NH];
#pragma unroll
    for (int q = 0; q < NH; ++q) acc[q] = 0.0f;
    auto drain = [&](int jc) {  // add chunk jc's accumulator
        const uint32_t col = (uint32_t)((jc & 1) * N + half * NH);
#pragma unroll
        for (int c = 0; c < NH; c += 8) {
            uint32_t v[8];
            const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + col + (uint32_t)c;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]),
                           "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[c + q] += __uint_as_float(v[q]);
        }
    };
    for (int j = 0; j < nchunk; ++j) {
        const int sidx = j & 1;
        float *aH = sm + sidx * STAGE, *aL = aH + 128 * 32, *bH = aL + 128 * 32, *bL = bH + N * 32;
        // the MMAs of chunk j-2 read this stage and wrote accumulator j & 1:
        // wait for them, then fold that accumulator into the registers
        if (j >= 2) {
            mbar_wait(&bar[sidx], ((j - 2) >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            drain(j - 2);
        }
        const int i = 16 * half;
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
            const float4 h4 = make_float4(tf32r(R.a[q]), tf32r(R.a[q + 1]), tf32r(R.a[q + 2]),
                                          tf32r(R.a[q + 3]));
            const float4 l4 = make_float4(tf32r(R.a[q] - h4.x), tf32r(R.a[q + 1] - h4.y),
                                          tf32r(R.a[q + 2] - h4.z), tf32r(R.a[q + 3] - h4.w));
            *reinterpret_cast<float4 *>(aH + swz(row, i + q)) = h4;
            *reinterpret_cast<float4 *>(aL + swz(row, i + q)) = l4;
        }
#pragma unroll
        for (int u = 0; u < ChunkRegs<N>::BPT; ++u) {
            const int e = tid + 256 * u;
            if (e < N * 32) {
                const int r = e >> 5, kk = e & 31;
                bH[swz(r, kk)] = R.bh[u];
                bL[swz(r, kk)] = R.bl[u];
            }
        }
        if (j + 1 < nchunk)
            load_chunk<N>(R, j + 1, half, tid, live, x, y, z, h, w, l, n, ic, K27, Kp, in, bhi,
                          blo);
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t tacc = tmem + (uint32_t)(sidx * N);
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint64_t ah = desc_swz(su32(aH) + 32 * s), al = desc_swz(su32(aL) + 32 * s);
                const uint64_t bh = desc_swz(su32(bH) + 32 * s), bl = desc_swz(su32(bL) + 32 * s);
                mma(tacc, ah, bh, id, s ? 1u : 0u);
                mma(tacc, ah, bl, id, 1u);
                mma(tacc, al, bh, id, 1u);
            }
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    su32(&bar[sidx])));
        }
    }
    // the last two chunks' accumulators
    for (int jc = (nchunk >= 2 ? nchunk - 2 : 0); jc < nchunk; ++jc) {
        mbar_wait(&bar[jc & 1], (jc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        drain(jc);
    }
    // epilogue: warps w and w+4 hold the two column halves of voxel row
    if (live)
#pragma unroll
        for (int q = 0; q < NH; ++q) {
            const int c = half * NH + q;
            out[(int64_t)c * n + p] = acc[q] + (bias ? bias[c] : 0.0f);
        }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(NCOL));
}

}  // namespace

extern "C" int tcconv_fwd(const float *in, int ic, int h, int w, int l, const float *wt,
                          const float *bias, int oc, float *out, float *scratch, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int Kp = (27 * ic + 31) / 32 * 32;
    float *bhi = scratch, *blo = scratch + (size_t)oc * Kp;
    prep_b<<<(oc * Kp + 255) / 256, 256, 0, st>>>(wt, oc, ic, Kp, bhi, blo);
    const int64_t n = (int64_t)h * w * l;
    const unsigned g = (unsigned)((n + 127) / 128);
    const size_t smem = (size_t)2 * (2 * 128 * 32 + 2 * oc * 32) * 4 + 1024;
#define TC(NV)                                                                                  \
    case NV:                                                                                    \
        cudaFuncSetAttribute(tcconv_k<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                             (int)smem);                                                        \
        tcconv_k<NV><<<g, 256, smem, st>>>(in, ic, h, w, l, bhi, blo, Kp, bias, out);           \
        break;
    if (ic % 16) return -1;  // the chunk loader assumes one tap per 16 channels
    switch (oc) {
        TC(8) TC(16) TC(32) TC(64) TC(128)
        default: return -1;
    }
#undef TC
    return (int)cudaPeekAtLastError();
}
