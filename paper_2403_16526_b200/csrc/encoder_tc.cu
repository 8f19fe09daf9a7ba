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
#include <cuda.h>
#include <cudaTypedefs.h>

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
            // lo = x - hi is exact in fp32; the MMA reads its top 19 bits (no second
            // rounding: the truncation error is 2^-21 |x|, far below the fp32 sums')
            const float4 l4 = make_float4(R.a[q] - h4.x, R.a[q + 1] - h4.y, R.a[q + 2] - h4.z,
                                          R.a[q + 3] - h4.w);
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

// ---------------------------------------------------------------------------
// Halo-tile form (volumes with h % 4 == 0, inputs with a multiple of 8
// channels): the CTA's 128 output voxels are an 8x4x4 block; per group of 8
// input channels one TMA box {24, 6, 6, 8} (x from x0-4, 1-voxel halo in y/z,
// zero fill outside the volume) lands in shared memory, double buffered, and
// the im2col K chunks are built from it (row pitch 24 floats: a warp's 8x4
// voxel reads hit 32 distinct banks).  Each input value is fetched once per
// CTA instead of once per tap.  K order: k = group * 224 + tap * 8 + c (27
// taps x 8 channels, padded to 7 chunks of 32 per group).
constexpr int HX = 24, HYZ = 6, HCG = 8, HPC = HX * HYZ * HYZ;  // floats per channel
constexpr int HGK = 224;                                         // K per channel group
constexpr int HBOX = HPC * HCG;                                  // floats per halo box

__global__ void prep_bh_k(const float *__restrict__ w, int oc, int ic, int flip, int nout, int N,
                          int Kin, float *__restrict__ bsw) {
    const int Kp = Kin / HCG * HGK;
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= nout * Kp) return;
    const int o = i / Kp, k = i % Kp;
    const int g = k / HGK, kl = k % HGK, tap = kl / HCG, c = g * HCG + kl % HCG;
    float v = 0.0f;
    if (tap < 27)
        v = flip ? w[((int64_t)c * ic + o) * 27 + (26 - tap)] : w[((int64_t)o * ic + c) * 27 + tap];
    const int nchunk = Kp / 32, z = o / N, r = o % N, j = k / 32, kk = k % 32;
    float *tile = bsw + (int64_t)((z * nchunk + j) * 2) * (N * 32);
    const float hv = tf32r(v);
    tile[swz(r, kk)] = hv;
    tile[N * 32 + swz(r, kk)] = tf32r(v - hv);
}

// HB halo buffers: 2 (prefetch the next group; one CTA per SM) or 1 (the box
// is reloaded after the group's last chunk; two CTAs per SM — the form used)
template <int N, int HB>
__global__ void __launch_bounds__(256, HB == 1 ? 2 : 1)
conv_halo_k(const __grid_constant__ CUtensorMap map, int Kin, int h, int w, int l,
            const float *__restrict__ bsw, int gsplit, int nout, const float *__restrict__ bias,
            int acc_out, float *__restrict__ out, float *__restrict__ part) {
    extern __shared__ __align__(1024) float sm_raw[];
    float *sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u) / 4;
    constexpr int STAGE = 2 * 128 * 32 + 2 * N * 32;
    constexpr int NH = N / 2;
    float *hs = sm + 2 * STAGE;  // two halo boxes
    __shared__ uint64_t bar[2], bbar[2], hbar[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int row = tid & 127, half = tid >> 7;
    const int ntx = (h + 7) / 8, nty = (w + 3) / 4;
    const int tz = blockIdx.x / (ntx * nty), rem = blockIdx.x - tz * ntx * nty;
    const int ty = rem / ntx, tx = rem - ty * ntx;
    const int x0 = tx * 8, y0 = ty * 4, z0 = tz * 4;
    const int rx = row & 7, ry = (row >> 3) & 3, rz = row >> 5;
    const int x = x0 + rx, y = y0 + ry, z = z0 + rz;
    const bool live = x < h && y < w && z < l;
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = ((int64_t)z * w + y) * h + x;
    constexpr uint32_t NCOL = 2 * N;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(&tmem_base)), "r"(NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bbar[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&hbar[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base, id = idesc_tf32(N);
    const int ngroups = Kin / HCG, nchunk = ngroups * (HGK / 32);
    const int gb = blockIdx.y * gsplit, ge = min(gb + gsplit, ngroups);
    const int cz = blockIdx.z * N;
    const float *btile = bsw + (int64_t)blockIdx.z * nchunk * 2 * (N * 32);
    auto issue_halo = [&](int g) {  // thread 0: group g's box into buffer g % HB
        uint64_t *mb = &hbar[g % HB];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)),
                     "r"((unsigned)(HBOX * sizeof(float)))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(su32(hs + (g % HB) * HBOX)),
            "l"(&map), "r"(x0 - 4), "r"(y0 - 1), "r"(z0 - 1), "r"(g * HCG), "r"(su32(mb))
            : "memory");
    };
    if (tid == 0) {
        issue_halo(gb);
        if (HB == 2 && gb + 1 < ge) issue_halo(gb + 1);
    }
    float acc[NH];
#pragma unroll
    for (int q = 0; q < NH; ++q) acc[q] = 0.0f;
    auto drain = [&](int tc) {
        const uint32_t col = (uint32_t)((tc & 1) * N + half * NH);
        uint32_t v[NH];
#pragma unroll
        for (int c = 0; c < NH; c += 8) {
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
    // this thread's voxel inside a halo box (tap (0,0,0) at dz = dy = dx = 0)
    const int hbase = (rz + 1) * (HYZ * HX) + (ry + 1) * HX + rx + 4;
    int t = 0;  // local chunk counter
    for (int g = gb; g < ge; ++g) {
        // (HB == 1: every thread is past the previous group's last barrier,
        // so its reads of the single box are done)
        if (tid == 0 && g > gb && (HB == 1 || g + 1 < ge)) issue_halo(HB == 1 ? g : g + 1);
        mbar_wait(&hbar[g % HB], (HB == 1 ? g - gb : (g - gb) >> 1) & 1);
        const float *hb = hs + (g % HB) * HBOX;
        for (int cc = 0; cc < HGK / 32; ++cc, ++t) {
            const int j = g * (HGK / 32) + cc, sidx = t & 1;
            float *aH = sm + sidx * STAGE, *aL = aH + 128 * 32, *bH = aL + 128 * 32,
                  *bL = bH + N * 32;
            if (t >= 2) {
                mbar_wait(&bar[sidx], ((t - 2) >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                drain(t - 2);
            }
            if (tid == 0)
                bulk_g2s(su32(bH), btile + (int64_t)j * 2 * (N * 32), 2 * N * 32 * 4, &bbar[sidx]);
            // 16 values: taps kt, kt + 1 (8 channels each) of this voxel
            const int kt = (cc * 32 + 16 * half) / HCG;
            float a[16];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int tap = kt + u;
                if (tap < 27) {
                    const int off = hbase + (tap / 9 - 1) * (HYZ * HX) + ((tap / 3) % 3 - 1) * HX +
                                    (tap % 3 - 1);
#pragma unroll
                    for (int c = 0; c < HCG; ++c) a[u * 8 + c] = hb[c * HPC + off];
                } else {
#pragma unroll
                    for (int c = 0; c < HCG; ++c) a[u * 8 + c] = 0.0f;
                }
            }
            const int i0 = 16 * half;
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
                const float4 h4 = make_float4(tf32r(a[q]), tf32r(a[q + 1]), tf32r(a[q + 2]),
                                              tf32r(a[q + 3]));
                const float4 l4 = make_float4(a[q] - h4.x, a[q + 1] - h4.y, a[q + 2] - h4.z,
                                              a[q + 3] - h4.w);  // (as in conv_k)
                *reinterpret_cast<float4 *>(aH + swz(row, i0 + q)) = h4;
                *reinterpret_cast<float4 *>(aL + swz(row, i0 + q)) = l4;
            }
            asm volatile("fence.proxy.async.shared::cta;");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();
            if (tid == 0) {
                mbar_wait(&bbar[sidx], (t >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t tacc = tmem + (uint32_t)(sidx * N);
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const uint64_t ah = desc_swz(su32(aH) + 32 * s),
                                   al = desc_swz(su32(aL) + 32 * s);
                    const uint64_t bh = desc_swz(su32(bH) + 32 * s),
                                   bl = desc_swz(su32(bL) + 32 * s);
                    mma(tacc, ah, bh, id, s ? 1u : 0u);
                    mma(tacc, ah, bl, id, 1u);
                    mma(tacc, al, bh, id, 1u);
                }
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        su32(&bar[sidx])));
            }
        }
    }
    const int nl = t;
    for (int tc = nl >= 2 ? nl - 2 : 0; tc < nl; ++tc) {
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

template <int N, int HB>
constexpr size_t halo_smem_bytes() {
    return (size_t)(2 * (2 * 128 * 32 + 2 * N * 32) + HB * HBOX) * sizeof(float) + 1024;
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

// MDG_ENC_TCH=0 turns the halo-tile form off (A/B comparisons)
static bool tch_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("MDG_ENC_TCH");
        return !(e && e[0] == '0');
    }();
    return on;
}

static PFN_cuTensorMapEncodeTiled_v12000 tc_tmap_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}

// the halo-tile form's tensor map; false when TMA cannot take the volume
// (row pitch not a multiple of 16 B, misaligned base, channels not in 8s)
static bool halo_map(CUtensorMap *map, const float *in, int kin, mdg_dims3 d) {
    if (!tch_enabled() || d.h % 4 != 0 || kin % tc::HCG != 0 ||
        reinterpret_cast<uintptr_t>(in) % 16 != 0 || !tc_tmap_fn())
        return false;
    const cuuint64_t dims[4] = {(cuuint64_t)d.h, (cuuint64_t)d.w, (cuuint64_t)d.l,
                                (cuuint64_t)kin};
    const cuuint64_t strides[3] = {(cuuint64_t)d.h * 4, (cuuint64_t)d.h * d.w * 4,
                                   (cuuint64_t)nvox(d) * 4};
    const cuuint32_t box[4] = {tc::HX, tc::HYZ, tc::HYZ, tc::HCG};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return tc_tmap_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(in), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static mdg_status enc_tc_halo(const CUtensorMap &map, int kin, mdg_dims3 d, const float *w,
                              int nout, int flip, const float *bias, bool acc, float *out,
                              cudaStream_t st) {
    const int64_t n = nvox(d);
    const int ngroups = kin / tc::HCG, Kp = ngroups * tc::HGK;
    const int N = 32, nz = 1;
    const int tiles = ((d.h + 7) / 8) * ((d.w + 3) / 4) * ((d.l + 3) / 4);
    // split the channel groups until the grid covers the GPU (2 CTAs per SM)
    int S = std::max(1, (2 * 148 + tiles * nz - 1) / (tiles * nz));
    S = std::min(S, ngroups);
    const int gsplit = (ngroups + S - 1) / S;
    S = (ngroups + gsplit - 1) / gsplit;
    Scratch sb;
    MDG_CUDA_TRY(sb.alloc(((size_t)2 * nout * Kp + (S > 1 ? (size_t)S * nout * n : 0)) *
                              sizeof(float), st));
    float *bsw = sb.as<float>();
    float *part = S > 1 ? bsw + (size_t)2 * nout * Kp : nullptr;
    const int wic = flip ? nout : kin, woc = flip ? kin : nout;
    tc::prep_bh_k<<<(nout * Kp + 255) / 256, 256, 0, st>>>(w, woc, wic, flip, nout, N, kin, bsw);
    MDG_LAUNCHED();
    const dim3 g((unsigned)tiles, (unsigned)S, (unsigned)nz);
    const int accf = acc ? 1 : 0;
    constexpr size_t sm = tc::halo_smem_bytes<32, 1>();
    MDG_CUDA_TRY(cudaFuncSetAttribute(tc::conv_halo_k<32, 1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    tc::conv_halo_k<32, 1><<<g, 256, sm, st>>>(map, kin, d.h, d.w, d.l, bsw, gsplit, nout, bias,
                                               accf, out, part);
    MDG_LAUNCHED();
    if (S > 1) {
        tc::split_reduce_k<<<(unsigned)(((int64_t)nout * n + 255) / 256), 256, 0, st>>>(
            part, S, nout, n, bias, accf, out);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

// out[o] (=, or += with acc) conv(in {kin, n}, B) for nout = 32, 64 or 128
// output channels.  flip = 0: the forward (w {nout, kin, 27}); flip = 1: the
// input gradient of a conv with weights w {kin, nout, 27} (gout has kin
// channels).  Small grids split K across CTAs (fixed-order reduction) and
// 128 outputs run as two 64-channel slices.
mdg_status enc_tc_conv(const float *in, int kin, mdg_dims3 d, const float *w, int nout, int flip,
                       const float *bias, bool acc, float *out, cudaStream_t st) {
    // 32 outputs: the halo-tile form (the 64-output one, at one CTA per SM,
    // measured slower than conv_k: 89 vs 77 us at L3 64->64)
    CUtensorMap hmap;
    if (nout == 32 && halo_map(&hmap, in, kin, d))
        return enc_tc_halo(hmap, kin, d, w, nout, flip, bias, acc, out, st);
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
