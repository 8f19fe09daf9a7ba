// encoder_igemm.cu — the encoder's conv3 (op_conv3d, ops.hpp:137-238) as an
// implicit GEMM on the FP32 pipe, for the deep pyramid levels whose volumes are
// too small to fill the GPU with the tiled slab kernel of encoder.cu.
//
//   out[o][p] (+)= sum_{c,t} wT[c][t][o] * in[c][p + off(t)]        (fwd / bwd_in)
//   gk[o][c][t]  += sum_p gout[o][p] * in[c][p + off(t)]             (wgrad)
//
// fwd / bwd_in: M = voxels (flattened p, so no tile is wasted on a 10-wide
// volume), N = output channels, K = input channels x 27 taps.  One CTA owns a
// BM x BN tile (BM * BN = 8192); each thread an 8-voxel x 4-channel register
// tile on the packed FP32 pipe (16 FFMA2 per 3 LDS.128 per tap).  K streams one
// input channel per stage through a cp.async double buffer: the 27 x BM
// im2col column gathered with zero fill at the volume faces, and the 27 x BN
// weight rows.  When the tile grid is small the input channels split across
// CTAs (split-K); the partials are summed in a fixed order by a second kernel
// (deterministic).
//
// wgrad: M = output channels, N = (input channel, tap), K = voxels; the same
// register tiling with gout^T and the im2col rows staged per 32-voxel step,
// voxels split across CTAs, fixed-order reduction of the per-CTA tiles.
#include <algorithm>

#include "mdg_common.cuh"

namespace mdg {
namespace enc {
namespace {

__device__ __forceinline__ unsigned sa(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cpa4(float *dst, const float *src, bool pred) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa(dst)), "l"(src),
                 "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cpa16(float *dst, const float *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct DI {
    int h, w, l, n, hw;
};

constexpr int NT = 256, TM = 8, TN = 4;

// fwd / bwd_in tile: BM = 256 voxels (one gathering thread per voxel, taps
// unrolled at compile time) x BN output channels; thread tile 8 voxels x FTN
// channels (FTN = 8 for BN = 64: 32 FFMA2 per 4 LDS.128 per tap)
template <int BN>
struct FTile {
    static constexpr int BM = NT, FTM = 8, FTN = BN >= 64 ? 8 : 4;
    static constexpr int WTN = BN / FTN;      // lanes along N per warp (8)
    static constexpr int WTM = 32 / WTN;      // lanes along M per warp (4)
    static constexpr int WM = BM / (FTM * WTM);
    static constexpr int ROW = BM + BN;       // floats per staged tap row
    static constexpr int STAGE = 27 * ROW;    // one input channel
    static_assert(WTN * WTM == 32 && WM * (BN / (FTN * WTN)) == NT / 32, "tile");
};

// ------------------------------------------------------------ fwd / bwd_in
template <int BN>
__global__ void __launch_bounds__(NT, 2)
igemm_fwd_k(const float *__restrict__ in, int cin, DI d, const float *__restrict__ wT, int opad,
            const float *__restrict__ bias, int cout, int acc_out, int cps,
            float *__restrict__ out, float *__restrict__ part) {
    using T = FTile<BN>;
    constexpr int FTM = T::FTM, FTN = T::FTN;
    extern __shared__ __align__(16) float smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int p0 = blockIdx.x * T::BM, n0 = blockIdx.y * BN;
    const int cb = blockIdx.z * cps, ce = min(cin, cb + cps);

    // gather role: this thread's voxel; the 27 taps' validity as one mask
    const int gp = p0 + tid;
    unsigned vm = 0;
    if (gp < d.n) {
        const int z = gp / d.hw, r = gp - z * d.hw, y = r / d.h, x = r - y * d.h;
        const unsigned mx = (x > 0 ? 1u : 0u) | 2u | (x < d.h - 1 ? 4u : 0u);
        const unsigned my = (y > 0 ? 1u : 0u) | 2u | (y < d.w - 1 ? 4u : 0u);
        const unsigned mz = (z > 0 ? 1u : 0u) | 2u | (z < d.l - 1 ? 4u : 0u);
#pragma unroll
        for (int dz = 0; dz < 3; ++dz)
#pragma unroll
            for (int dy = 0; dy < 3; ++dy)
                if ((mz >> dz) & (my >> dy) & 1u) vm |= mx << (dz * 9 + dy * 3);
    }
    auto stage = [&](int c, float *buf) {
        const float *src = in + (int64_t)c * d.n + gp;
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            const int off = (t / 9 - 1) * d.hw + ((t / 3) % 3 - 1) * d.h + (t % 3 - 1);
            const bool ok = (vm >> t) & 1u;
            cpa4(buf + t * T::ROW + tid, ok ? src + off : in, ok);
        }
        const float *wr = wT + (int64_t)c * 27 * opad + n0;
        for (int i = tid; i < 27 * (BN / 4); i += NT) {
            const int t = i / (BN / 4), j = (i - t * (BN / 4)) * 4;
            cpa16(buf + t * T::ROW + T::BM + j, wr + (int64_t)t * opad + j);
        }
        cp_commit();
    };

    const int lm = lane % T::WTM, ln = lane / T::WTM;
    const int wm = wid % T::WM, wn = wid / T::WM;
    const int m0 = (wm * T::WTM + lm) * FTM, nn0 = (wn * T::WTN + ln) * FTN;
    float2 acc[FTM][FTN / 2];
#pragma unroll
    for (int i = 0; i < FTM; ++i)
#pragma unroll
        for (int j = 0; j < FTN / 2; ++j) acc[i][j] = make_float2(0.0f, 0.0f);

    if (cb < ce) stage(cb, smem);
    for (int c = cb; c < ce; ++c) {
        float *cur = smem + ((c - cb) & 1) * T::STAGE;
        if (c + 1 < ce) {
            stage(c + 1, smem + ((c + 1 - cb) & 1) * T::STAGE);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
#pragma unroll 3
        for (int t = 0; t < 27; ++t) {
            const float *row = cur + t * T::ROW;
            const float4 a0 = *reinterpret_cast<const float4 *>(row + m0);
            const float4 a1 = *reinterpret_cast<const float4 *>(row + m0 + 4);
            float2 b2[FTN / 2];
#pragma unroll
            for (int q = 0; q < FTN / 4; ++q) {
                const float4 b = *reinterpret_cast<const float4 *>(row + T::BM + nn0 + 4 * q);
                b2[2 * q] = make_float2(b.x, b.y);
                b2[2 * q + 1] = make_float2(b.z, b.w);
            }
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
            for (int i = 0; i < FTM; ++i) {
                const float2 ai = make_float2(av[i], av[i]);
#pragma unroll
                for (int j = 0; j < FTN / 2; ++j) acc[i][j] = __ffma2_rn(ai, b2[j], acc[i][j]);
            }
        }
        __syncthreads();
    }

    // epilogue
#pragma unroll
    for (int j = 0; j < FTN; ++j) {
        const int o = n0 + nn0 + j;
        if (o >= cout) continue;
        const float bo = (part || acc_out || !bias) ? 0.0f : bias[o];
        float *dst = part ? part + ((int64_t)blockIdx.z * cout + o) * d.n : out + (int64_t)o * d.n;
#pragma unroll
        for (int i = 0; i < FTM; ++i) {
            const int p = p0 + m0 + i;
            if (p < d.n) {
                const float v = (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x;
                if (part)
                    dst[p] = v;
                else
                    dst[p] = acc_out ? dst[p] + v : bo + v;
            }
        }
    }
}

// out[o][p] (+)= [bias[o]] + sum_z part[z][o][p]   (fixed z order)
__global__ void __launch_bounds__(256)
igemm_splitk_sum_k(const float *__restrict__ part, int nsplit, int cout, int n,
                   const float *__restrict__ bias, int acc_out, float *__restrict__ out) {
    const int64_t total = (int64_t)cout * n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        float v = 0.0f;
        for (int z = 0; z < nsplit; ++z) v += part[(int64_t)z * total + i];
        const int o = (int)(i / n);
        out[i] = acc_out ? out[i] + v : (bias ? bias[o] : 0.0f) + v;
    }
}

template <int BN>
cudaError_t launch_fwd(const float *in, int cin, DI d, const float *wT, int opad,
                       const float *bias, int cout, bool acc_out, float *out, cudaStream_t st) {
    using T = FTile<BN>;
    const int mt = (d.n + T::BM - 1) / T::BM, nt = (cout + BN - 1) / BN;
    const int tiles = mt * nt;
    const int want = 148 * 2 * 2;  // ~2 waves at 2 CTAs/SM, >= 8 channels per split
    int nsplit = std::max(1, std::min(std::max(1, cin / 8), (want + tiles - 1) / tiles));
    const int cps = (cin + nsplit - 1) / nsplit;
    nsplit = (cin + cps - 1) / cps;
    const size_t smem = 2 * (size_t)T::STAGE * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(igemm_fwd_k<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    Scratch part;
    if (nsplit > 1) {
        e = part.alloc((size_t)nsplit * cout * d.n * sizeof(float), st);
        if (e != cudaSuccess) return e;
    }
    igemm_fwd_k<BN><<<dim3(mt, nt, nsplit), NT, smem, st>>>(
        in, cin, d, wT, opad, bias, cout, acc_out ? 1 : 0, cps, out,
        nsplit > 1 ? part.as<float>() : nullptr);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if ((e = cudaPeekAtLastError()) != cudaSuccess) return e;
    if (nsplit > 1) {
        const int64_t total = (int64_t)cout * d.n;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
        igemm_splitk_sum_k<<<blocks, 256, 0, st>>>(part.as<float>(), nsplit, cout, d.n, bias,
                                                   acc_out ? 1 : 0, out);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if ((e = cudaPeekAtLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ------------------------------------------------------------------ wgrad
// part[kb][o][ct] = sum_{p in chunk kb} gout[o][p] * in[c][p + off(t)],
// ct = c*27 + t; partb[kb][o] = sum gout[o][p] (bias gradient, N-tile 0 only).
constexpr int WBK = 32;  // voxels per stage

template <int BM>  // output channels per CTA (M), BN = 8192 / BM (ct)
__global__ void __launch_bounds__(NT, 2)
igemm_wgrad_k(const float *__restrict__ in, int cin, DI d, const float *__restrict__ gout,
              int cout, int chunk, float *__restrict__ part, float *__restrict__ partb) {
    constexpr int BN = NT * TM * TN / BM;  // 128 (BM 64) / 256 (BM 32)
    constexpr int WTN = 8, WTM = 4;        // lanes: 4 along M (TM=8 ch), 8 along N (TN=4 ct)
    constexpr int WM = BM / (TM * WTM);    // warps along M
    constexpr int AROW = BM + 4, BROW = BN + 4;
    constexpr int STAGE = WBK * (AROW + BROW);
    static_assert((BM / TM) * (BN / TN) == NT, "tile");
    extern __shared__ __align__(16) float smem[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int kb = blockIdx.x, o0 = blockIdx.y * BM, ct0 = blockIdx.z * BN;
    const int nct = cin * 27;
    const int pb = kb * chunk, pe = min(d.n, pb + chunk);

    // gather roles: lane = voxel within the step; warp wid -> rows wid + 8k.
    // Row offsets and taps are step-invariant; per step only the voxel's
    // 27-bit face mask changes.
    constexpr int KB = BN / 8;
    int roff[KB];
    unsigned char rtap[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) {
        const int ct = ct0 + wid + 8 * k;
        const int c = ct / 27, t = ct - c * 27;
        roff[k] = c * d.n + (t / 9 - 1) * d.hw + ((t / 3) % 3 - 1) * d.h + (t % 3 - 1);
        rtap[k] = ct < nct ? (unsigned char)t : (unsigned char)31;  // 31: never valid
    }
    auto stage = [&](int ps, float *buf) {
        const int p = ps + lane;
        unsigned vm = 0;
        if (p < pe) {
            const int z = p / d.hw, r = p - z * d.hw, y = r / d.h, x = r - y * d.h;
            const unsigned mx = (x > 0 ? 1u : 0u) | 2u | (x < d.h - 1 ? 4u : 0u);
            const unsigned my = (y > 0 ? 1u : 0u) | 2u | (y < d.w - 1 ? 4u : 0u);
            const unsigned mz = (z > 0 ? 1u : 0u) | 2u | (z < d.l - 1 ? 4u : 0u);
#pragma unroll
            for (int dz = 0; dz < 3; ++dz)
#pragma unroll
                for (int dy = 0; dy < 3; ++dy)
                    if ((mz >> dz) & (my >> dy) & 1u) vm |= mx << (dz * 9 + dy * 3);
        }
        float *As = buf, *Bs = buf + WBK * AROW;
#pragma unroll
        for (int k = 0; k < BM / 8; ++k) {
            const int o = wid + 8 * k;
            const bool ok = vm != 0 && o0 + o < cout;
            cpa4(As + lane * AROW + o, ok ? gout + (int64_t)(o0 + o) * d.n + p : gout, ok);
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const bool ok = (vm >> rtap[k]) & 1u;
            cpa4(Bs + lane * BROW + wid + 8 * k, ok ? in + (p + roff[k]) : in, ok);
        }
        cp_commit();
    };

    const int lm = lane % WTM, ln = lane / WTM;
    const int wm = wid % WM, wn = wid / WM;
    const int m0 = (wm * WTM + lm) * TM, nn0 = (wn * WTN + ln) * TN;
    float2 acc[TM][TN / 2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN / 2; ++j) acc[i][j] = make_float2(0.0f, 0.0f);
    float bsum = 0.0f;

    const int nsteps = (pe - pb + WBK - 1) / WBK;
    if (nsteps > 0) stage(pb, smem);
    for (int s = 0; s < nsteps; ++s) {
        float *cur = smem + (s & 1) * STAGE;
        if (s + 1 < nsteps) {
            stage(pb + (s + 1) * WBK, smem + ((s + 1) & 1) * STAGE);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const float *As = cur, *Bs = cur + WBK * AROW;
#pragma unroll 8
        for (int q = 0; q < WBK; ++q) {
            const float4 a0 = *reinterpret_cast<const float4 *>(As + q * AROW + m0);
            const float4 a1 = *reinterpret_cast<const float4 *>(As + q * AROW + m0 + 4);
            const float4 b = *reinterpret_cast<const float4 *>(Bs + q * BROW + nn0);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float2 b01 = make_float2(b.x, b.y), b23 = make_float2(b.z, b.w);
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const float2 ai = make_float2(av[i], av[i]);
                acc[i][0] = __ffma2_rn(ai, b01, acc[i][0]);
                acc[i][1] = __ffma2_rn(ai, b23, acc[i][1]);
            }
        }
        if (blockIdx.z == 0 && tid < BM)
            for (int q = 0; q < WBK; ++q) bsum += As[q * AROW + tid];
        __syncthreads();
    }
    float *dst = part + (((int64_t)kb * gridDim.y + blockIdx.y) * gridDim.z + blockIdx.z) * (BM * BN);
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN / 2; ++j)
            *reinterpret_cast<float2 *>(dst + (m0 + i) * BN + nn0 + 2 * j) = acc[i][j];
    if (blockIdx.z == 0 && tid < BM) partb[((int64_t)kb * gridDim.y + blockIdx.y) * BM + tid] = bsum;
}

// gk[o][c][t] += sum_kb part[kb][tile(o, ct)][...]; gb[o] += sum_kb partb.
// One thread per output value walking the partials in kb order (fixed order;
// consecutive threads read consecutive addresses of each partial tile).
template <int BM>
__global__ void __launch_bounds__(256)
igemm_wgrad_sum_k(const float *__restrict__ part, const float *__restrict__ partb, int nkb,
                  int nmy, int nnz, int cout, int cin, float *__restrict__ gk,
                  float *__restrict__ gb) {
    constexpr int BN = NT * TM * TN / BM;
    const int nct = cin * 27, nw = cout * nct;
    const int idx = blockIdx.x * 256 + threadIdx.x;
    if (idx >= nw + cout) return;
    float v = 0.0f;
    if (idx < nw) {
        const int o = idx / nct, ct = idx - o * nct;
        const int my = o / BM, ol = o - my * BM, nz = ct / BN, cl = ct - nz * BN;
        const float *src = part + ((int64_t)(my * nnz + nz) * BM + ol) * BN + cl;
        const int64_t stride = (int64_t)nmy * nnz * BM * BN;
#pragma unroll 4
        for (int b = 0; b < nkb; ++b) v += src[b * stride];
        if (gk) gk[idx] += v;
    } else {
        const int o = idx - nw, my = o / BM, ol = o - my * BM;
        for (int b = 0; b < nkb; ++b) v += partb[((int64_t)b * nmy + my) * BM + ol];
        if (gb) gb[o] += v;
    }
}

template <int BM>
cudaError_t launch_wgrad(const float *in, int cin, DI d, const float *gout, int cout, float *gk,
                         float *gb, cudaStream_t st) {
    constexpr int BN = NT * TM * TN / BM;
    constexpr int STAGE = WBK * ((BM + 4) + (BN + 4));
    const int nmy = (cout + BM - 1) / BM, nnz = (cin * 27 + BN - 1) / BN;
    const int tiles = nmy * nnz;
    const int want = 148 * 2 * 2;  // ~2 waves, >= 8 voxel steps per CTA
    int nkb = std::max(1, (want + tiles - 1) / tiles);
    int chunk = (d.n + nkb - 1) / nkb;
    chunk = std::max(WBK * 8, (chunk + WBK - 1) / WBK * WBK);
    nkb = (d.n + chunk - 1) / chunk;
    const size_t smem = 2 * (size_t)STAGE * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(igemm_wgrad_k<BM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    Scratch part;
    const size_t np = (size_t)nkb * tiles * BM * BN;
    if ((e = part.alloc((np + (size_t)nkb * nmy * BM) * sizeof(float), st)) != cudaSuccess) return e;
    float *pb = part.as<float>() + np;
    igemm_wgrad_k<BM><<<dim3(nkb, nmy, nnz), NT, smem, st>>>(in, cin, d, gout, cout, chunk,
                                                             part.as<float>(), pb);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if ((e = cudaPeekAtLastError()) != cudaSuccess) return e;
    const int nout = cout * cin * 27 + cout;
    igemm_wgrad_sum_k<BM><<<(nout + 255) / 256, 256, 0, st>>>(part.as<float>(), pb, nkb, nmy,
                                                              nnz, cout, cin, gk, gb);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaPeekAtLastError();
}

}  // namespace

// out (+)= conv(in) with prepared weights wT[c][t][opad] (opad a multiple of
// the chosen N tile).  Returns false if this path does not take the shape.
int igemm_fwd_bn(int cout) { return cout > 32 ? 64 : 32; }

mdg_status igemm_conv_fwd(const float *in, int cin, mdg_dims3 dd, const float *wT, int opad,
                          const float *bias, int cout, bool acc_out, float *out,
                          cudaStream_t st) {
    const DI d{dd.h, dd.w, dd.l, dd.h * dd.w * dd.l, dd.h * dd.w};
    const cudaError_t e = igemm_fwd_bn(cout) == 64
                              ? launch_fwd<64>(in, cin, d, wT, opad, bias, cout, acc_out, out, st)
                              : launch_fwd<32>(in, cin, d, wT, opad, bias, cout, acc_out, out, st);
    return e == cudaSuccess ? MDG_OK : status_from_cuda(e, "igemm_conv_fwd");
}

mdg_status igemm_conv_wgrad(const float *in, int cin, mdg_dims3 dd, const float *gout, int cout,
                            float *gk, float *gb, cudaStream_t st) {
    const DI d{dd.h, dd.w, dd.l, dd.h * dd.w * dd.l, dd.h * dd.w};
    const cudaError_t e = cout > 32 ? launch_wgrad<64>(in, cin, d, gout, cout, gk, gb, st)
                                    : launch_wgrad<32>(in, cin, d, gout, cout, gk, gb, st);
    return e == cudaSuccess ? MDG_OK : status_from_cuda(e, "igemm_conv_wgrad");
}

}  // namespace enc
}  // namespace mdg
