// encoder_tc.cu — the encoder's 3x3x3 convolution (ops.hpp:58-99, zero padded)
// on the 5th-generation tensor cores, for the levels where that wins: 32, 64
// and 128 output channels (L2-L4 of the small preset), forward and input
// gradient.
//
// Implicit GEMM D[voxel][o] = sum_k A[voxel][k] B[o][k], k = tap * ic + c:
//   * one CTA = 128 consecutive output voxels (the MMA's M) and 256 threads:
//     thread pairs gather their voxel's 32-value K chunk (im2col on the fly,
//     one tap x 16 channels each), with the NEXT chunk's global loads in
//     flight while this one is split and stored; the chunk's weight tiles
//     (pre-split, pre-swizzled) arrive by one bulk copy;
//   * fp32 accuracy from 3xTF32: every operand is split into tf32 hi + lo,
//     stored 128-byte swizzled K-major in shared memory; one thread issues
//     4 K-steps x (hi*hi + hi*lo + lo*hi) = 12 tcgen05.mma per chunk;
//   * each chunk accumulates into a FRESH TMEM accumulator (two, alternating)
//     and the chunk sums are added in fp32 registers (round to nearest, in
//     chunk order): the tensor core never accumulates across chunks, which
//     keeps the error at ~2e-7 relative to float64 (a single TMEM accumulator
//     over 100+ K steps drifts to 1e-5; tools/exp/tcconv.cu);
//   * two shared-memory stages; chunk j's operands are free when the commit
//     of chunk j-2 has arrived on its mbarrier.
// The input gradient is the same convolution of gout with the flipped,
// transposed kernel (w'[c][o][26 - t] = w[o][c][t]).  Measured against the
// FFMA2 / implicit-GEMM kernels it replaces: 1.2-1.8x faster
// at these shapes and about 3x more accurate; slower for N <= 16, which keeps
// the old kernels.  Grids too small to fill the GPU split K across CTAs.
#include <algorithm>
#include <cstdlib>

#include "mdg_common.cuh"

namespace mdg {
namespace tc {

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// element (r, k) of an R x 32 fp32 tile, 128-byte swizzle (8-row atoms of 1 KB)
__device__ __forceinline__ int swz(int r, int k) {
    return ((r >> 3) * 1024 + (r & 7) * 128 + (((k >> 2) ^ (r & 7)) << 4)) / 4 + (k & 3);
}
// shared-memory matrix descriptor: K-major, SWIZZLE_128B, 1 KB between 8-row atoms
__device__ __forceinline__ uint64_t desc_swz(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) |
           ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: D f32, A / B tf32, both K-major, M = 128
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

// B = the weights as {nout, Kp} (k = tap * ic + c, zero padded to Kp), split
// into tf32 hi / lo and stored as the shared-memory image of each (N-slice z,
// chunk j): tile ((z * nchunk + j) * 2 + {0: hi, 1: lo}) of N x 32 floats in
// the 128-byte-swizzled order, so one bulk copy stages a chunk's B.
// flip: the input-gradient kernel w'[c][o][26 - t] of w {oc, ic, 27}
__global__ void prep_b_k(const float *__restrict__ w, int oc, int ic, int flip, int nout, int N,
                         int Kin, int Kp, float *__restrict__ bsw) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= nout * Kp) return;
    const int o = i / Kp, k = i % Kp;
    float v = 0.0f;
    if (k < 27 * Kin) {
        const int tap = k / Kin, c = k % Kin;
        v = flip ? w[((int64_t)c * ic + o) * 27 + (26 - tap)] : w[((int64_t)o * ic + c) * 27 + tap];
    }
    const int nchunk = Kp / 32, z = o / N, r = o % N, j = k / 32, kk = k % 32;
    float *tile = bsw + (int64_t)((z * nchunk + j) * 2) * (N * 32);
    const float h = tf32r(v);
    tile[swz(r, kk)] = h;
    tile[N * 32 + swz(r, kk)] = tf32r(v - h);
}

struct ChunkRegs {
    float a[16];
};

// this thread's share of the next K chunk: 16 channels (c0 ..) of one tap of
// its voxel (Kin % 16 == 0, so a half chunk never straddles taps); tap / c0
// advance by 32 values per chunk
__device__ __forceinline__ void load_chunk(ChunkRegs &R, int &tap, int &c0, bool live, int x, int y,
                                           int z, int h, int w, int l, int64_t n, int Kin,
                                           const float *__restrict__ in) {
    bool ok = false;
    int64_t off = 0;
    if (tap < 27 && live) {
        const int xx = x + tap % 3 - 1, yy = y + (tap / 3) % 3 - 1, zz = z + tap / 9 - 1;
        ok = xx >= 0 && xx < h && yy >= 0 && yy < w && zz >= 0 && zz < l;
        off = (int64_t)c0 * n + ((int64_t)zz * w + yy) * h + xx;
    }
    const float *src = in + off;
#pragma unroll
    for (int q = 0; q < 16; ++q) R.a[q] = ok ? __ldg(src + (int64_t)q * n) : 0.0f;
    c0 += 32;
    while (c0 >= Kin) {
        c0 -= Kin;
        ++tap;
    }
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}

// blockIdx.x: 128-voxel tile; blockIdx.y: K split (chunks [y*jsplit, ..));
// blockIdx.z: the output-channel slice [z*N, z*N+N) of nout.  With part
// non-null the split's partial sums go to part[y][c][p] (the reduce kernel
// adds them in split order); otherwise out (=, or += with acc_out) + bias.
template <int N>
__global__ void __launch_bounds__(256)
conv_k(const float *__restrict__ in, int Kin, int h, int w, int l, const float *__restrict__ bsw,
       int Kp, int jsplit, int nout,
       const float *__restrict__ bias, int acc_out, float *__restrict__ out,
       float *__restrict__ part) {
    extern __shared__ __align__(1024) float sm_raw[];
    // the swizzle atoms start on 1 KB boundaries of the shared window
    float *sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u) / 4;
    constexpr int STAGE = 2 * 128 * 32 + 2 * N * 32;  // floats per stage
    constexpr int NH = N / 2;
    __shared__ uint64_t bar[2], bbar[2];  // MMA commits; B bulk copies
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int row = tid & 127, half = tid >> 7;  // voxel row; K half / column half
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
    constexpr uint32_t NCOL = 2 * N;  // two accumulators (64 or 128 columns)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(&tmem_base)), "r"(NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base, id = idesc_tf32(N);
    const int jb = blockIdx.y * jsplit, je = min(jb + jsplit, Kp / 32), nl = je - jb;
    const int cz = blockIdx.z * N;  // first output channel of this CTA
    const int nchunk = Kp / 32;
    const float *btile = bsw + (int64_t)blockIdx.z * nchunk * 2 * (N * 32);
    float acc[NH];
#pragma unroll
    for (int q = 0; q < NH; ++q) acc[q] = 0.0f;
    // fold chunk jc's accumulator into the registers: warps w and w + 4 read
    // TMEM lanes 32 (w % 4) .. +31, column halves [0, N/2) and [N/2, N)
    auto drain = [&](int tc) {  // local chunk index: accumulator tc & 1
        const uint32_t col = (uint32_t)((tc & 1) * N + half * NH);
        uint32_t v[NH];
#pragma unroll
        for (int c = 0; c < NH; c += 8) {  // all loads in flight, one wait
            const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + col + (uint32_t)c;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[c]), "=r"(v[c + 1]), "=r"(v[c + 2]), "=r"(v[c + 3]),
                           "=r"(v[c + 4]), "=r"(v[c + 5]), "=r"(v[c + 6]), "=r"(v[c + 7])
                         : "r"(taddr));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int q = 0; q < NH; ++q) acc[q] += __uint_as_float(v[q]);
    };
    ChunkRegs R;
    int tap, c0;
    {
        const int k0 = 32 * jb + 16 * half;
        tap = k0 < 27 * Kin ? k0 / Kin : 27;
        c0 = k0 - tap * Kin;
    }
    load_chunk(R, tap, c0, live, x, y, z, h, w, l, n, Kin, in);
    for (int t = 0; t < nl; ++t) {  // local chunk t = global chunk jb + t
        const int j = jb + t, sidx = t & 1;
        float *aH = sm + sidx * STAGE, *aL = aH + 128 * 32, *bH = aL + 128 * 32, *bL = bH + N * 32;
        if (t >= 2) {  // chunk t-2's MMAs read this stage and wrote accumulator t & 1
            mbar_wait(&bar[sidx], ((t - 2) >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            drain(t - 2);
        }
        if (tid == 0)  // this chunk's B (hi and lo tiles, contiguous) by one bulk copy
            bulk_g2s(su32(bH), btile + (int64_t)j * 2 * (N * 32), 2 * N * 32 * 4, &bbar[sidx]);
        const int i0 = 16 * half;
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
            const float4 h4 = make_float4(tf32r(R.a[q]), tf32r(R.a[q + 1]), tf32r(R.a[q + 2]),
                                          tf32r(R.a[q + 3]));
            const float4 l4 = make_float4(tf32r(R.a[q] - h4.x), tf32r(R.a[q + 1] - h4.y),
                                          tf32r(R.a[q + 2] - h4.z), tf32r(R.a[q + 3] - h4.w));
            *reinterpret_cast<float4 *>(aH + swz(row, i0 + q)) = h4;
            *reinterpret_cast<float4 *>(aL + swz(row, i0 + q)) = l4;
        }
        if (t + 1 < nl)  // the next chunk's loads fly during the handoff below
            load_chunk(R, tap, c0, live, x, y, z, h, w, l, n, Kin, in);
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (tid == 0) {
            mbar_wait(&bbar[sidx], (t >> 1) & 1);
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
    for (int tc = nl >= 2 ? nl - 2 : 0; tc < nl; ++tc) {  // the last two chunks
        mbar_wait(&bar[tc & 1], (tc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        drain(tc);
    }
    if (live) {
        if (part) {
#pragma unroll
            for (int q = 0; q < NH; ++q)
                part[((int64_t)blockIdx.y * nout + cz + half * NH + q) * n + p] = acc[q];
        } else {
#pragma unroll
            for (int q = 0; q < NH; ++q) {
                const int c = cz + half * NH + q;
                float *o = out + (int64_t)c * n + p;
                const float v = acc[q] + (bias ? bias[c] : 0.0f);
                *o = acc_out ? *o + v : v;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(NCOL));
}

// out[c][p] (=, or +=) sum over splits s in order of part[s][c][p], + bias
__global__ void split_reduce_k(const float *__restrict__ part, int S, int nout, int64_t n,
                               const float *__restrict__ bias, int acc_out,
                               float *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= (int64_t)nout * n) return;
    const int c = (int)(i / n);
    float v = 0.0f;
    for (int s = 0; s < S; ++s) v += part[(int64_t)s * nout * n + i];
    v += bias ? bias[c] : 0.0f;
    out[i] = acc_out ? out[i] + v : v;
}

template <int N>
constexpr size_t smem_bytes() {
    return (size_t)2 * (2 * 128 * 32 + 2 * N * 32) * sizeof(float) + 1024;
}

}  // namespace tc

// MDG_ENC_TC=0 turns the tensor-core path off (A/B comparisons)
static bool tc_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("MDG_ENC_TC");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool enc_tc_conv_ok(int kin, int nout, mdg_dims3 d) {
    const int64_t n = (int64_t)d.h * d.w * d.l;
    return tc_enabled() && (nout == 32 || nout == 64 || nout == 128) && kin % 16 == 0 &&
           kin <= 128 && n >= 128 && n < (int64_t(1) << 31);
}

// out[o] (=, or += with acc) conv(in {kin, n}, B) for nout = 32, 64 or 128
// output channels.  flip = 0: the forward (w {nout, kin, 27}); flip = 1: the
// input gradient of a conv with weights w {kin, nout, 27} (gout has kin
// channels).  Small grids split K across CTAs (fixed-order reduction) and
// 128 outputs run as two 64-channel slices.
mdg_status enc_tc_conv(const float *in, int kin, mdg_dims3 d, const float *w, int nout, int flip,
                       const float *bias, bool acc, float *out, cudaStream_t st) {
    const int Kp = (27 * kin + 31) / 32 * 32, nchunk = Kp / 32;
    const int N = nout == 32 ? 32 : 64, nz = nout / N;
    const int64_t n = (int64_t)d.h * d.w * d.l;
    const int tiles = (int)((n + 127) / 128);
    // enough CTAs for 2 per SM, each split >= 4 chunks
    int S = std::max(1, (2 * 148 + tiles * nz - 1) / (tiles * nz));
    S = std::min(S, std::max(1, nchunk / 4));
    const int jsplit = (nchunk + S - 1) / S;
    S = (nchunk + jsplit - 1) / jsplit;
    Scratch sb;
    MDG_CUDA_TRY(sb.alloc(((size_t)2 * nout * Kp + (S > 1 ? (size_t)S * nout * n : 0)) *
                              sizeof(float), st));
    float *bsw = sb.as<float>();
    float *part = S > 1 ? bsw + (size_t)2 * nout * Kp : nullptr;
    // w's ic (the forward's input channels): kin forward, nout for the flip
    const int wic = flip ? nout : kin, woc = flip ? kin : nout;
    tc::prep_b_k<<<(nout * Kp + 255) / 256, 256, 0, st>>>(w, woc, wic, flip, nout, N, kin, Kp,
                                                          bsw);
    MDG_LAUNCHED();
    const dim3 g((unsigned)tiles, (unsigned)S, (unsigned)nz);
    const int accf = acc ? 1 : 0;
    if (N == 32) {
        constexpr size_t sm = tc::smem_bytes<32>();
        MDG_CUDA_TRY(cudaFuncSetAttribute(tc::conv_k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sm));
        tc::conv_k<32><<<g, 256, sm, st>>>(in, kin, d.h, d.w, d.l, bsw, Kp, jsplit, nout, bias,
                                           accf, out, part);
    } else {
        constexpr size_t sm = tc::smem_bytes<64>();
        MDG_CUDA_TRY(cudaFuncSetAttribute(tc::conv_k<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sm));
        tc::conv_k<64><<<g, 256, sm, st>>>(in, kin, d.h, d.w, d.l, bsw, Kp, jsplit, nout, bias,
                                           accf, out, part);
    }
    MDG_LAUNCHED();
    if (S > 1) {
        tc::split_reduce_k<<<(unsigned)(((int64_t)nout * n + 255) / 256), 256, 0, st>>>(
            part, S, nout, n, bias, accf, out);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

}  // namespace mdg
