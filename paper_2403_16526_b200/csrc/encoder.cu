// encoder.cu — the feature encoder's kernels on sm_100a:
// conv blocks (conv3 -> InstanceNorm -> LeakyReLU, twice) and 2x average
// pooling (encoder.hpp:87-116, ops.hpp:58-99, 137-238, sampling.hpp:171-219).
//
// conv3 (any ic -> oc): one CTA computes a 32x8x4 voxel block for 8 output
// channels.  Input channels stream through shared memory four at a time (the
// 6x10x34 slab with a zero halo, batched loads), the weights of the chunk sit
// in shared memory as [ci][tap][oc] so each tap is one broadcast float2-pair
// read, and every thread accumulates its 4 voxels x 8 channels on the packed
// FP32 pipe (FFMA2 with a broadcast input value).  The input gradient is the
// same kernel with the flipped, transposed kernel and accumulation into the
// existing gradient; the kernel gradient is a per-block outer-product sum
// over shared-memory tiles with a fixed-order cross-block reduction.
// Accumulation is FMA-contracted: results match the CPU reference to fp32
// tolerance (tests: relative norm 1e-4).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "mdg_common.cuh"

namespace mdg {
namespace enc {

constexpr int TX = 32, TY = 8, TV = 4;               // voxel block
constexpr int HX = TX + 2, HY = TY + 2, HZ = TV + 2;  // slab with halo
constexpr int SLAB = HZ * HY * HX;                    // one channel
constexpr int CIB = 4;                                // input channels per stage
constexpr int OCB = 8;                                // output channels per CTA
constexpr int NT = TX * TY;

struct D3 {
    int h, w, l, n;
};

// input channels [c0, c0+nch) of `src`, planes z0-1 .. z0+TV, rows y0-1 ..,
// columns x0-1 .., zero outside the volume; all loads issued before stores
template <int MAXCH>
__device__ __forceinline__ void stage1(float *dst, const float *__restrict__ src, int nch,
                                       const D3 &d, int x0, int y0, int z0) {
    constexpr int kRows = HZ * HY;
    constexpr int kIt = (MAXCH * kRows + 7) / 8;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gx0 = x0 - 1 + lane, gx1 = x0 + 31 + lane;
    const bool okx0 = gx0 >= 0 && gx0 < d.h, okx1 = lane < 2 && gx1 < d.h;
    float v0[kIt], v1[kIt];
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
        const int r = wid + 8 * it;
        v0[it] = v1[it] = 0.0f;
        if (r < nch * kRows) {
            const int c = r / kRows, rr = r - c * kRows;
            const int dz = rr / HY, yy = rr - dz * HY;
            const int gy = y0 - 1 + yy, gz = z0 - 1 + dz;
            if (gy >= 0 && gy < d.w && gz >= 0 && gz < d.l) {
                const float *row = src + (int64_t)c * d.n + ((int64_t)gz * d.w + gy) * d.h;
                if (okx0) v0[it] = __ldg(row + gx0);
                if (okx1) v1[it] = __ldg(row + gx1);
            }
        }
    }
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
        const int r = wid + 8 * it;
        if (r < nch * kRows) {
            dst[r * HX + lane] = v0[it];
            if (lane < 2) dst[r * HX + 32 + lane] = v1[it];
        }
    }
}

// up to CIB channels, two at a time (bounded register window)
__device__ __forceinline__ void stage(float *dst, const float *__restrict__ src, int nch,
                                      const D3 &d, int x0, int y0, int z0) {
    for (int c = 0; c < nch; c += 2)
        stage1<2>(dst + c * SLAB, src + (int64_t)c * d.n, min(2, nch - c), d, x0, y0, z0);
}

// wT[c][t][o] (o padded to a multiple of OCB with zeros) from the reference
// layout w[oc][ic][27]:  fwd: c = ci, o = co, tap t;  flip (input gradient):
// c = co, o = ci, tap 26 - t
__global__ void wprep_k(const float *__restrict__ w, int oc, int ic, int flip, int opad,
                        float *__restrict__ wT) {
    const int cin = flip ? oc : ic, cout = flip ? ic : oc;
    const int total = cin * 27 * opad;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int o = i % opad, t = (i / opad) % 27, c = i / (27 * opad);
        float v = 0.0f;
        if (o < cout) v = flip ? w[((int64_t)c * ic + o) * 27 + (26 - t)] : w[((int64_t)o * ic + c) * 27 + t];
        wT[i] = v;
    }
}

// out[o][p] (+)= bias[o] + sum_c sum_t wT[c][t][o] * in[c][p + off(t)]
template <bool ACC>
__global__ void __launch_bounds__(NT, 2)
conv3g_k(const float *__restrict__ in, int cin, D3 d, const float *__restrict__ wT, int opad,
         const float *__restrict__ bias, int cout, float *__restrict__ out) {
    __shared__ __align__(16) float slab[CIB * SLAB];
    __shared__ __align__(16) float ws[CIB * 27 * OCB];
    const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
    const int nzb = (d.l + TV - 1) / TV;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = blockIdx.z % nzb, ob = blockIdx.z / nzb;
    const int z0 = zb * TV, o0 = ob * OCB;
    float2 acc[TV][OCB / 2];
#pragma unroll
    for (int j = 0; j < OCB / 2; ++j) {
        const float b0 = (!ACC && bias && o0 + 2 * j < cout) ? bias[o0 + 2 * j] : 0.0f;
        const float b1 = (!ACC && bias && o0 + 2 * j + 1 < cout) ? bias[o0 + 2 * j + 1] : 0.0f;
#pragma unroll
        for (int v = 0; v < TV; ++v) acc[v][j] = make_float2(b0, b1);
    }
    const float *tp = slab + ty * HX + tx;
    for (int c0 = 0; c0 < cin; c0 += CIB) {
        const int nch = min(CIB, cin - c0);
        __syncthreads();
        stage(slab, in + (int64_t)c0 * d.n, nch, d, x0, y0, z0);
        for (int i = threadIdx.x; i < nch * 27 * OCB; i += NT) {
            const int c = i / (27 * OCB), r = i - c * 27 * OCB;
            ws[i] = wT[((int64_t)(c0 + c) * 27) * opad + (r / OCB) * opad + o0 + (r % OCB)];
        }
        __syncthreads();
        for (int c = 0; c < nch; ++c) {
            const float *sp = tp + c * SLAB;
            const float4 *wc = reinterpret_cast<const float4 *>(ws + c * 27 * OCB);
#pragma unroll
            for (int t = 0; t < 27; ++t) {
                const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
                const float4 wa = wc[2 * t], wb = wc[2 * t + 1];
                const float2 w2[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w),
                                      make_float2(wb.x, wb.y), make_float2(wb.z, wb.w)};
#pragma unroll
                for (int v = 0; v < TV; ++v) {
                    const float xv = sp[((v + dz) * HY + dy) * HX + dx];
                    const float2 x2 = make_float2(xv, xv);
#pragma unroll
                    for (int j = 0; j < OCB / 2; ++j) acc[v][j] = __ffma2_rn(x2, w2[j], acc[v][j]);
                }
            }
        }
    }
    const int x = x0 + tx, y = y0 + ty;
    if (x >= d.h || y >= d.w) return;
#pragma unroll
    for (int v = 0; v < TV; ++v) {
        const int z = z0 + v;
        if (z >= d.l) break;
        const int64_t p = ((int64_t)z * d.w + y) * d.h + x;
#pragma unroll
        for (int j = 0; j < OCB / 2; ++j) {
            const int o = o0 + 2 * j;
            if (o < cout) {
                float *q = out + (int64_t)o * d.n + p;
                *q = ACC ? *q + acc[v][j].x : acc[v][j].x;
            }
            if (o + 1 < cout) {
                float *q = out + (int64_t)(o + 1) * d.n + p;
                *q = ACC ? *q + acc[v][j].y : acc[v][j].y;
            }
        }
    }
}

// per channel: Chan's parallel combination (in double, fixed tile order) of
// the per-tile (sum, M2) pairs -> mean[c] and inv[c] = 1/sqrt(var + eps),
// var = M2 / n (op_instance_norm ops.hpp:170-181: biased variance)
__global__ void __launch_bounds__(256)
in_stats_k(const float2 *__restrict__ stats, D3 d, int ntx, int nty, int ntz, float eps,
           float *__restrict__ mean, float *__restrict__ inv) {
    const int c = blockIdx.x, ntiles = ntx * nty * ntz;
    const float2 *st = stats + (int64_t)c * ntiles;
    double n = 0.0, mu = 0.0, m2 = 0.0;
    for (int t = threadIdx.x; t < ntiles; t += 256) {
        const int bx = t % ntx, by = (t / ntx) % nty, bz = t / (ntx * nty);
        const double nb = (double)min(TX, d.h - bx * TX) * min(TY, d.w - by * TY) *
                          min(TV, d.l - bz * TV);
        const float2 v = st[t];
        const double mb = (double)v.x / nb, tot = n + nb, dl = mb - mu;
        mu += dl * nb / tot;
        m2 += (double)v.y + dl * dl * n * nb / tot;
        n = tot;
    }
    __shared__ double sn[256], smu[256], sm2[256];
    sn[threadIdx.x] = n;
    smu[threadIdx.x] = mu;
    sm2[threadIdx.x] = m2;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            const double na = sn[threadIdx.x], nb = sn[threadIdx.x + h], tot = na + nb;
            if (nb > 0.0) {
                const double dl = smu[threadIdx.x + h] - smu[threadIdx.x];
                smu[threadIdx.x] += dl * nb / tot;
                sm2[threadIdx.x] += sm2[threadIdx.x + h] + dl * dl * na * nb / tot;
                sn[threadIdx.x] = tot;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        mean[c] = (float)smu[0];
        inv[c] = 1.0f / sqrtf((float)(sm2[0] / sn[0]) + eps);
    }
}

// ---- TMA-staged variant (h % 4 == 0, 16-B aligned planes): the chunk's
// slab is ONE 4-D box load {40, 10, 6, CIB} (x0-4 .. x0+35 so the start is
// 16-B aligned; faces and missing channels zero-filled by the TMA unit) and
// its weights one bulk copy from the blocked layout wB[ob][c][t][8]; two
// buffers on mbarriers, so staging costs the threads nothing and overlaps
// the previous chunk's FMAs.
constexpr int PX = 40, XO = 3;            // TMA row pitch, offset of x0-1
constexpr int SLABT = HZ * HY * PX;       // one channel
constexpr int WCH = 27 * OCB;             // weights of one input channel
constexpr int TBUF = CIB * SLABT + CIB * WCH;  // floats per stage buffer
constexpr size_t TSMEM = (2 * (size_t)TBUF + 8) * sizeof(float);

__device__ __forceinline__ unsigned s32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void t_wait(uint64_t *b, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(s32(b)), "r"(phase)
            : "memory");
    } while (!done);
}

template <bool ACC>
__global__ void __launch_bounds__(NT, 2)
conv3t_k(const __grid_constant__ CUtensorMap map, int cin, D3 d, const float *__restrict__ wB,
         int cpad, const float *__restrict__ bias, int cout, float *__restrict__ out,
         float2 *__restrict__ stats) {
    extern __shared__ __align__(128) float tsm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(tsm + 2 * TBUF);
    const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
    const int nzb = (d.l + TV - 1) / TV;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = blockIdx.z % nzb, ob = blockIdx.z / nzb;
    const int z0 = zb * TV, o0 = ob * OCB;
    const int nck = (cin + CIB - 1) / CIB;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int k) {
        float *b = tsm + (k & 1) * TBUF;
        uint64_t *mb = &bar[k & 1];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s32(mb)),
                     "r"((unsigned)(TBUF * sizeof(float)))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(s32(b)),
            "l"(&map), "r"(x0 - 4), "r"(y0 - 1), "r"(z0 - 1), "r"(k * CIB), "r"(s32(mb))
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];\n" ::"r"(s32(b + CIB * SLABT)),
            "l"(wB + ((int64_t)ob * cpad + k * CIB) * WCH), "r"((unsigned)(CIB * WCH * sizeof(float))),
            "r"(s32(mb))
            : "memory");
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (nck > 1) issue(1);
    }
    float2 acc[TV][OCB / 2];
#pragma unroll
    for (int j = 0; j < OCB / 2; ++j) {
        const float b0 = (!ACC && bias && o0 + 2 * j < cout) ? bias[o0 + 2 * j] : 0.0f;
        const float b1 = (!ACC && bias && o0 + 2 * j + 1 < cout) ? bias[o0 + 2 * j + 1] : 0.0f;
#pragma unroll
        for (int v = 0; v < TV; ++v) acc[v][j] = make_float2(b0, b1);
    }
    for (int k = 0; k < nck; ++k) {
        const float *b = tsm + (k & 1) * TBUF;
        t_wait(&bar[k & 1], (k >> 1) & 1);
        const int nch = min(CIB, cin - k * CIB);
        const float *tp = b + ty * PX + tx + XO;
        for (int c = 0; c < nch; ++c) {
            const float *sp = tp + c * SLABT;
            const float4 *wc = reinterpret_cast<const float4 *>(b + CIB * SLABT + c * WCH);
#pragma unroll
            for (int t = 0; t < 27; ++t) {
                const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
                const float4 wa = wc[2 * t], wb = wc[2 * t + 1];
                const float2 w2[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w),
                                      make_float2(wb.x, wb.y), make_float2(wb.z, wb.w)};
#pragma unroll
                for (int v = 0; v < TV; ++v) {
                    const float xv = sp[((v + dz) * HY + dy) * PX + dx];
                    const float2 x2 = make_float2(xv, xv);
#pragma unroll
                    for (int j = 0; j < OCB / 2; ++j) acc[v][j] = __ffma2_rn(x2, w2[j], acc[v][j]);
                }
            }
        }
        __syncthreads();  // every warp is done with buffer k & 1
        if (threadIdx.x == 0 && k + 2 < nck) issue(k + 2);
    }
    const int x = x0 + tx, y = y0 + ty;
    if (!ACC && stats) {
        // InstanceNorm statistics of this tile per output channel: the sum,
        // then M2 about the tile mean (two block reductions); the per-tile
        // (sum, M2) pairs are combined in a fixed order by in_stats_k
        __shared__ float red[8][OCB];
        __shared__ float tmean[OCB];
        const int nx = min(TX, d.h - x0), ny = min(TY, d.w - y0), nz = min(TV, d.l - z0);
        const float cnt = (float)(nx * ny * nz);
        const bool inxy = x < d.h && y < d.w;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        float s[OCB];
#pragma unroll
        for (int j = 0; j < OCB; ++j) s[j] = 0.0f;
#pragma unroll
        for (int v = 0; v < TV; ++v)
            if (inxy && z0 + v < d.l)
#pragma unroll
                for (int j = 0; j < OCB / 2; ++j) {
                    s[2 * j] += acc[v][j].x;
                    s[2 * j + 1] += acc[v][j].y;
                }
#pragma unroll
        for (int j = 0; j < OCB; ++j) {
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], m);
            if (lane == 0) red[wid][j] = s[j];
        }
        __syncthreads();
        if (threadIdx.x < OCB) {
            float a = 0.0f;
#pragma unroll
            for (int w8 = 0; w8 < 8; ++w8) a += red[w8][threadIdx.x];
            tmean[threadIdx.x] = a / cnt;
            s[0] = a;  // keep the sum for the write below
        }
        __syncthreads();
        float q[OCB];
#pragma unroll
        for (int j = 0; j < OCB; ++j) q[j] = 0.0f;
#pragma unroll
        for (int v = 0; v < TV; ++v)
            if (inxy && z0 + v < d.l)
#pragma unroll
                for (int j = 0; j < OCB / 2; ++j) {
                    const float a = acc[v][j].x - tmean[2 * j], b = acc[v][j].y - tmean[2 * j + 1];
                    q[2 * j] = fmaf(a, a, q[2 * j]);
                    q[2 * j + 1] = fmaf(b, b, q[2 * j + 1]);
                }
        float sum_keep = s[0];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < OCB; ++j) {
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) q[j] += __shfl_xor_sync(0xffffffffu, q[j], m);
            if (lane == 0) red[wid][j] = q[j];
        }
        __syncthreads();
        if (threadIdx.x < OCB && o0 + threadIdx.x < cout) {
            float m2 = 0.0f;
#pragma unroll
            for (int w8 = 0; w8 < 8; ++w8) m2 += red[w8][threadIdx.x];
            const int ntiles = gridDim.x * gridDim.y * ((d.l + TV - 1) / TV);
            const int tile = (zb * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            stats[(int64_t)(o0 + threadIdx.x) * ntiles + tile] = make_float2(sum_keep, m2);
        }
    }
    if (x >= d.h || y >= d.w) return;
#pragma unroll
    for (int v = 0; v < TV; ++v) {
        const int z = z0 + v;
        if (z >= d.l) break;
        const int64_t p = ((int64_t)z * d.w + y) * d.h + x;
#pragma unroll
        for (int j = 0; j < OCB / 2; ++j) {
            const int o = o0 + 2 * j;
            if (o < cout) {
                float *q = out + (int64_t)o * d.n + p;
                *q = ACC ? *q + acc[v][j].x : acc[v][j].x;
            }
            if (o + 1 < cout) {
                float *q = out + (int64_t)(o + 1) * d.n + p;
                *q = ACC ? *q + acc[v][j].y : acc[v][j].y;
            }
        }
    }
}

// blocked weights for conv3t_k: wB[ob][c][t][j] = w of output ob*8+j, input c
// (c < cpad, zero-padded), tap t; flip as wprep_k
__global__ void wprep_blocked_k(const float *__restrict__ w, int oc, int ic, int flip, int cpad,
                                int nob, float *__restrict__ wB) {
    const int cin = flip ? oc : ic, cout = flip ? ic : oc;
    const int total = nob * cpad * WCH;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int j = i % OCB, t = (i / OCB) % 27, c = (i / WCH) % cpad, ob = i / (WCH * cpad);
        const int o = ob * OCB + j;
        float v = 0.0f;
        if (o < cout && c < cin)
            v = flip ? w[((int64_t)c * ic + o) * 27 + (26 - t)] : w[((int64_t)o * ic + c) * 27 + t];
        wB[i] = v;
    }
}

// ---- TMA-staged kernel gradient for narrow outputs (cout <= 16 per pass of
// 8).  gk[o][c][t] = sum_p gout[o][p] * in[c][p + off(t)].  A CTA owns a 32x8
// x-y tile, a z range, 8 output channels and WC input channels; each z step
// stages ZW planes of gout ({32, 8, ZW, 8} box) and ZW+2 planes of input
// ({40, 10, ZW+2, WC} box, faces zero-filled) by TMA into a double buffer.
// Warp (c, dz), lane x: per voxel it reads one new input row triple (the
// y-sliding window keeps the other two) and the 8 gout values, and issues
// 36 FFMA2 into 9 taps x 8 channels of register accumulators.  Zero fill
// makes out-of-volume voxels contribute exactly 0, so there are no bounds
// checks.  At the end each warp reduces its 72 sums across lanes (fixed
// butterfly) into a per-CTA partial; a fixed-order pass adds the partials.
constexpr int ZW = 4;
template <int WC, int OH = 1>  // OH: output-channel halves per (c, dz) warp
struct WT {
    static constexpr int IN = WC * (ZW + 2) * HY * PX;  // input floats per stage
    static constexpr int GO = OCB * ZW * TY * TX;         // gout floats per stage
    static constexpr int BUF = IN + GO;
    static constexpr size_t SMEM = (2 * (size_t)BUF + 8) * sizeof(float);
    static constexpr int NTH = 3 * WC * 32 * OH;
    static constexpr int OPW = OCB / OH;  // output channels per warp
};

template <int WC, int OH = 1>
__global__ void __launch_bounds__(3 * WC * 32 * OH)
conv3w_k(const __grid_constant__ CUtensorMap imap, const __grid_constant__ CUtensorMap gmap,
         int cin, int cout, D3 d, int zper, int ncc, float *__restrict__ part,
         float *__restrict__ partb) {
    using W = WT<WC, OH>;
    constexpr int PJ = W::OPW / 2;  // channel pairs per warp
    extern __shared__ __align__(128) float wsm2[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(wsm2 + 2 * W::BUF);
    int *cnt = reinterpret_cast<int *>(wsm2 + 2 * W::BUF + 4);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int hh = wid % OH, cl = wid / (3 * OH), dz = (wid / OH) % 3;
    const int ob0 = hh * W::OPW;  // this warp's first output channel (in the block of 8)
    // grid x = (x-y tile, channel chunk) with the chunk fastest: the chunks of
    // one tile run side by side and share its gout planes through L2
    const int ntx = (d.h + TX - 1) / TX;
    const int cc = blockIdx.x % ncc, txy = blockIdx.x / ncc;
    const int x0 = (txy % ntx) * TX, y0 = (txy / ntx) * TY;
    const int zb0 = blockIdx.y * zper, zb1 = min(d.l, zb0 + zper);
    const int ob = blockIdx.z;
    const int c0 = cc * WC;
    const int nsteps = (zb1 - zb0 + ZW - 1) / ZW;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        cnt[0] = cnt[1] = 0;
    }
    __syncthreads();
    auto issue = [&](int k) {
        float *b = wsm2 + (k & 1) * W::BUF;
        uint64_t *mb = &bar[k & 1];
        const int z = zb0 + k * ZW;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s32(mb)),
                     "r"((unsigned)(W::BUF * sizeof(float)))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(s32(b)),
            "l"(&imap), "r"(x0 - 4), "r"(y0 - 1), "r"(z - 1), "r"(c0), "r"(s32(mb))
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(s32(b + W::IN)),
            "l"(&gmap), "r"(x0), "r"(y0), "r"(z), "r"(ob * OCB), "r"(s32(mb))
            : "memory");
    };
    if (threadIdx.x == 0) {
        if (nsteps > 0) issue(0);
        if (nsteps > 1) issue(1);
    }
    float2 acc[9][PJ];
#pragma unroll
    for (int k = 0; k < 9; ++k)
#pragma unroll
        for (int j = 0; j < PJ; ++j) acc[k][j] = make_float2(0.0f, 0.0f);
    // bias gradient: in the first channel chunk, the warps of input channel 0
    // (dz = 0..2, each half) sum their pairs j with j % 3 == dz
    constexpr int NS = (PJ + 2) / 3;
    float2 gsum[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) gsum[q] = make_float2(0.0f, 0.0f);
    const bool bias_warp = cc == 0 && cl == 0;

    for (int k = 0; k < nsteps; ++k) {
        const float *b = wsm2 + (k & 1) * W::BUF;
        t_wait(&bar[k & 1], (k >> 1) & 1);
        if (c0 + cl < cin) {
#pragma unroll
            for (int v = 0; v < ZW; ++v) {
                const float *ip = b + ((cl * (ZW + 2) + v + dz) * HY) * PX + lane + XO;
                const float *gp = b + W::IN + (v * TY) * TX + lane;
                float r0[3], r1[3];
#pragma unroll
                for (int dx = 0; dx < 3; ++dx) {
                    r0[dx] = ip[dx];
                    r1[dx] = ip[PX + dx];
                }
#pragma unroll
                for (int y = 0; y < TY; ++y) {
                    float r2[3];
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx) r2[dx] = ip[(y + 2) * PX + dx];
                    float2 g2[PJ];
#pragma unroll
                    for (int j = 0; j < PJ; ++j)
                        g2[j] = make_float2(gp[(ob0 + 2 * j) * (ZW * TY * TX) + y * TX],
                                            gp[(ob0 + 2 * j + 1) * (ZW * TY * TX) + y * TX]);
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx) {
                        const float2 s0 = make_float2(r0[dx], r0[dx]);
                        const float2 s1 = make_float2(r1[dx], r1[dx]);
                        const float2 s2 = make_float2(r2[dx], r2[dx]);
#pragma unroll
                        for (int j = 0; j < PJ; ++j) {
                            acc[dx][j] = __ffma2_rn(s0, g2[j], acc[dx][j]);
                            acc[3 + dx][j] = __ffma2_rn(s1, g2[j], acc[3 + dx][j]);
                            acc[6 + dx][j] = __ffma2_rn(s2, g2[j], acc[6 + dx][j]);
                        }
                    }
                    if (bias_warp) {
#pragma unroll
                        for (int j = 0; j < PJ; ++j)
                            if (j % 3 == dz) gsum[j / 3] = __fadd2_rn(gsum[j / 3], g2[j]);
                    }
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx) {
                        r0[dx] = r1[dx];
                        r1[dx] = r2[dx];
                    }
                }
            }
        }
        // release the buffer without a block barrier: the last warp out
        // re-arms it with the step two ahead (warps drift within the slack)
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&cnt[k & 1], 1) == W::NTH / 32 - 1) {
                cnt[k & 1] = 0;
                __threadfence_block();
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                if (k + 2 < nsteps) issue(k + 2);
            }
        }
    }
    // per-CTA partial: part[((ob*ncc + cc)*nblk + blk)][o][c][t]
    const int nxy = gridDim.x / ncc;
    const int nblk = nxy * gridDim.y, blk = blockIdx.y * nxy + txy;
    float *dst = part + ((int64_t)(ob * ncc + cc) * nblk + blk) * (OCB * WC * 27);
#pragma unroll
    for (int k = 0; k < 9; ++k)
#pragma unroll
        for (int j = 0; j < PJ; ++j) {
            float ax = acc[k][j].x, ay = acc[k][j].y;
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) {
                ax += __shfl_xor_sync(0xffffffffu, ax, m);
                ay += __shfl_xor_sync(0xffffffffu, ay, m);
            }
            if (lane == 0) {
                const int t = dz * 9 + k;  // k = dy*3 + dx
                dst[((ob0 + 2 * j) * WC + cl) * 27 + t] = ax;
                dst[((ob0 + 2 * j + 1) * WC + cl) * 27 + t] = ay;
            }
        }
    if (bias_warp) {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            const int j = dz + 3 * q;
            if (j >= PJ) break;
            float ax = gsum[q].x, ay = gsum[q].y;
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) {
                ax += __shfl_xor_sync(0xffffffffu, ax, m);
                ay += __shfl_xor_sync(0xffffffffu, ay, m);
            }
            if (lane == 0) {
                partb[((int64_t)ob * nblk + blk) * OCB + ob0 + 2 * j] = ax;
                partb[((int64_t)ob * nblk + blk) * OCB + ob0 + 2 * j + 1] = ay;
            }
        }
    }
}

// gk[o][c][t] += sum_blk part; gb[o] += sum_blk partb (one warp per value,
// lanes stride the CTAs, fixed butterfly)
template <int WC>
__global__ void __launch_bounds__(256)
conv3w_sum_k(const float *__restrict__ part, const float *__restrict__ partb, int nblk, int ncc,
             int cout, int cin, float *__restrict__ gk, float *__restrict__ gb) {
    const int nw = cout * cin * 27;
    const int idx = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (idx >= nw + cout) return;
    float v = 0.0f;
    if (idx < nw) {
        const int o = idx / (cin * 27), c = (idx / 27) % cin, t = idx % 27;
        const int ob = o / OCB, ol = o % OCB, cc = c / WC, cw = c % WC;
        const float *src = part + (int64_t)(ob * ncc + cc) * nblk * (OCB * WC * 27) +
                           (ol * WC + cw) * 27 + t;
        for (int b = lane; b < nblk; b += 32) v += src[(int64_t)b * (OCB * WC * 27)];
    } else {
        const int o = idx - nw, ob = o / OCB, ol = o % OCB;
        for (int b = lane; b < nblk; b += 32) v += partb[((int64_t)ob * nblk + b) * OCB + ol];
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    if (lane == 0) {
        if (idx < nw) {
            if (gk) gk[idx] += v;
        } else if (gb) {
            gb[idx - nw] += v;
        }
    }
}

// kernel / bias gradient partials of one voxel block:
//   part[blk][o][c][t] = sum_p gout[o][p] * in[c][p + off(t)]   (o in the
//   CTA's 8-channel block, c in its 4-channel block), partb[blk][o] = sum gout.
// Lanes run along x (conflict-free shared-memory rows).  A warp owns kernel
// rows (c, dz, dy); per voxel row each lane loads the three input taps and the
// eight gout values of its column and accumulates 8 x 3 products (4 x 3 FFMA2
// on channel pairs); the warp reduces the 24 sums at the end of the row set.
constexpr int WG_NT = 288;  // 9 warps x 4 kernel rows = 36 = CIB * 9

__global__ void __launch_bounds__(WG_NT, 3)
conv3g_wgrad_k(const float *__restrict__ in, int cin, D3 d, const float *__restrict__ gout,
               int cout, float *__restrict__ part, float *__restrict__ partb) {
    extern __shared__ __align__(16) float wsm[];  // slab [CIB*SLAB] | gout tile [OCB][1024]
    float *slab = wsm;
    float(*gs)[TV * TY * TX] = reinterpret_cast<float(*)[TV * TY * TX]>(wsm + CIB * SLAB);
    const int ntx = (d.h + TX - 1) / TX, nty = (d.w + TY - 1) / TY;
    const int blk = blockIdx.x;
    const int bx = blk % ntx, by = (blk / ntx) % nty, bz = blk / (ntx * nty);
    const int x0 = bx * TX, y0 = by * TY, z0 = bz * TV;
    const int o0 = blockIdx.y * OCB, c0 = blockIdx.z * CIB;
    const int nch = min(CIB, cin - c0);
    if (threadIdx.x < NT) stage(slab, in + (int64_t)c0 * d.n, nch, d, x0, y0, z0);
    for (int i = threadIdx.x; i < OCB * TV * TY * TX; i += blockDim.x) {
        const int o = i / (TV * TY * TX), r = i - o * (TV * TY * TX);
        const int v = r / (TY * TX), yy = (r / TX) % TY, xx = r % TX;
        const int x = x0 + xx, y = y0 + yy, z = z0 + v;
        float g = 0.0f;
        if (o0 + o < cout && x < d.h && y < d.w && z < d.l)
            g = __ldg(gout + (int64_t)(o0 + o) * d.n + ((int64_t)z * d.w + y) * d.h + x);
        gs[o][r] = g;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *dstb = part + (((int64_t)blk * gridDim.y + blockIdx.y) * gridDim.z + blockIdx.z) *
                             (OCB * CIB * 27);
    for (int it = 0; it < 4; ++it) {
        const int row = wid * 4 + it;  // (c, dz, dy)
        const int c = row / 9, dz = (row % 9) / 3, dy = row % 3;
        float2 acc[3][OCB / 2];
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
            for (int j = 0; j < OCB / 2; ++j) acc[dx][j] = make_float2(0.0f, 0.0f);
        if (c < nch) {
            for (int vy = 0; vy < TV * TY; ++vy) {
                const int v = vy / TY, yy = vy % TY;
                const float *srow = slab + c * SLAB + ((v + dz) * HY + yy + dy) * HX + lane;
                const float sv[3] = {srow[0], srow[1], srow[2]};
                float2 g2[OCB / 2];
#pragma unroll
                for (int j = 0; j < OCB / 2; ++j)
                    g2[j] = make_float2(gs[2 * j][vy * TX + lane], gs[2 * j + 1][vy * TX + lane]);
#pragma unroll
                for (int dx = 0; dx < 3; ++dx) {
                    const float2 s2 = make_float2(sv[dx], sv[dx]);
#pragma unroll
                    for (int j = 0; j < OCB / 2; ++j) acc[dx][j] = __ffma2_rn(g2[j], s2, acc[dx][j]);
                }
            }
        }
        // warp reduction of the 24 sums (fixed butterfly order)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
            for (int j = 0; j < OCB / 2; ++j) {
                float ax = acc[dx][j].x, ay = acc[dx][j].y;
#pragma unroll
                for (int m = 16; m > 0; m >>= 1) {
                    ax += __shfl_xor_sync(0xffffffffu, ax, m);
                    ay += __shfl_xor_sync(0xffffffffu, ay, m);
                }
                if (lane == 0) {
                    const int t = dz * 9 + dy * 3 + dx;
                    dstb[((2 * j) * CIB + c) * 27 + t] = ax;
                    dstb[((2 * j + 1) * CIB + c) * 27 + t] = ay;
                }
            }
    }
    if (blockIdx.z == 0 && threadIdx.x < OCB) {
        float sb = 0.0f;
        for (int r = 0; r < TV * TY * TX; ++r) sb += gs[threadIdx.x][r];
        partb[((int64_t)blk * gridDim.y + blockIdx.y) * OCB + threadIdx.x] = sb;
    }
}

// fixed-order sum of the per-CTA partials into gk[o][c][t] (+=) and gb[o]
// for many partials: one 256-thread block per output value
__global__ void __launch_bounds__(256)
conv3g_wgrad_tree_k(const float *__restrict__ part, const float *__restrict__ partb, int nblk,
                    int noy, int ncz, int cout, int cin, float *__restrict__ gk,
                    float *__restrict__ gb) {
    const int idx = blockIdx.x;
    const int nw = cout * cin * 27;
    float v = 0.0f;
    if (idx < nw) {
        const int o = idx / (cin * 27), c = (idx / 27) % cin, t = idx % 27;
        const int oy = o / OCB, ol = o % OCB, cz = c / CIB, cl = c % CIB;
        for (int b = threadIdx.x; b < nblk; b += 256)
            v += part[(((int64_t)b * noy + oy) * ncz + cz) * (OCB * CIB * 27) + (ol * CIB + cl) * 27 + t];
    } else {
        const int o = idx - nw, oy = o / OCB, ol = o % OCB;
        for (int b = threadIdx.x; b < nblk; b += 256) v += partb[((int64_t)b * noy + oy) * OCB + ol];
    }
    __shared__ float sm[256];
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int m = 128; m > 0; m >>= 1) {
        if (threadIdx.x < m) sm[threadIdx.x] += sm[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (idx < nw) {
            if (gk) gk[idx] += sm[0];
        } else if (gb) {
            gb[idx - nw] += sm[0];
        }
    }
}

// few partials: one thread per output value
__global__ void __launch_bounds__(256)
conv3g_wgrad_final_k(const float *__restrict__ part, const float *__restrict__ partb, int nblk,
                     int noy, int ncz, int cout, int cin, float *__restrict__ gk,
                     float *__restrict__ gb) {
    const int idx = blockIdx.x * 256 + threadIdx.x;
    const int nw = cout * cin * 27;
    if (idx >= nw + cout) return;
    float v = 0.0f;
    if (idx < nw) {
        const int o = idx / (cin * 27), c = (idx / 27) % cin, t = idx % 27;
        const int oy = o / OCB, ol = o % OCB, cz = c / CIB, cl = c % CIB;
        for (int b = 0; b < nblk; ++b)
            v += part[(((int64_t)b * noy + oy) * ncz + cz) * (OCB * CIB * 27) + (ol * CIB + cl) * 27 + t];
        if (gk) gk[idx] += v;
    } else {
        const int o = idx - nw, oy = o / OCB, ol = o % OCB;
        for (int b = 0; b < nblk; ++b) v += partb[((int64_t)b * noy + oy) * OCB + ol];
        if (gb) gb[o] += v;
    }
}

// ------------------------------------------------ instance norm + leaky relu
// Channel-plane loops: one grid row per channel, float4 when n % 4 == 0 (the
// planes are then 16-B aligned), two loads in flight per thread.
template <bool VEC>
struct Plane {
    static constexpr int W = VEC ? 4 : 1;
};
__device__ __forceinline__ float4 ld4(const float *p, int i) {
    return reinterpret_cast<const float4 *>(p)[i];
}
__device__ __forceinline__ void st4(float *p, int i, float4 v) {
    reinterpret_cast<float4 *>(p)[i] = v;
}
__device__ __forceinline__ float el(const float4 &v, int k) {
    return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

template <int NV>
__device__ __forceinline__ void block_sum(float (&v)[NV], float *out) {
    __shared__ float red[NV][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], m);
        if (lane == 0) red[k][wid] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        float a = 0.0f;
#pragma unroll
        for (int w = 0; w < 8; ++w) a += red[threadIdx.x][w];
        out[threadIdx.x] = a;
    }
}

// per-channel partial sums (pass 1: x, pass 2: (x - mean)^2 with mean given)
template <bool VEC>
__global__ void __launch_bounds__(256)
chan_sum_k(const float *__restrict__ x, int n, const float *__restrict__ mean,
           float *__restrict__ part) {
    const int c = blockIdx.y;
    const float *src = x + (int64_t)c * n;
    const float mu = mean ? mean[c] : 0.0f;
    float a[1] = {0.0f};
    const int nv = VEC ? n >> 2 : n;
#pragma unroll 2
    for (int i = blockIdx.x * 256 + threadIdx.x; i < nv; i += gridDim.x * 256) {
        if (VEC) {
            const float4 v = ld4(src, i);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (mean) {
                    const float t = el(v, k) - mu;
                    a[0] = fmaf(t, t, a[0]);
                } else {
                    a[0] += el(v, k);
                }
            }
        } else {
            const float v = src[i];
            if (mean) {
                const float t = v - mu;
                a[0] = fmaf(t, t, a[0]);
            } else {
                a[0] += v;
            }
        }
    }
    block_sum<1>(a, part + (int64_t)c * gridDim.x + blockIdx.x);
}

// stat[c] = sum(part[c]) / n  (inv = 1: 1 / sqrt(. + eps); inv = 2: the raw
// sum, for a slab whose statistics are all-reduced); fixed order
__global__ void __launch_bounds__(256)
chan_final_k(const float *__restrict__ part, int nparts, int n, int inv, float eps,
             float *__restrict__ stat) {
    const int c = blockIdx.x;
    float v[1] = {0.0f};
    for (int i = threadIdx.x; i < nparts; i += 256) v[0] += part[(int64_t)c * nparts + i];
    __shared__ float r;
    block_sum<1>(v, &r);
    __syncthreads();
    if (threadIdx.x == 0) {
        const float m = r / (float)n;
        stat[c] = inv == 2 ? r : inv ? 1.0f / sqrtf(m + eps) : m;
    }
}

// z = lrelu(gamma (x - mean) inv + beta)   (ops.hpp:184-185, 230)
template <bool VEC>
__global__ void __launch_bounds__(256)
in_apply_k(const float *__restrict__ x, int n, const float *__restrict__ mean,
           const float *__restrict__ inv, const float *__restrict__ g,
           const float *__restrict__ b, float slope, float *__restrict__ z) {
    const int c = blockIdx.y;
    const float mu = mean[c], iv = inv[c], gg = g[c], bb = b[c];
    const float *src = x + (int64_t)c * n;
    float *dst = z + (int64_t)c * n;
    auto f = [&](float xv) {
        const float y = gg * (xv - mu) * iv + bb;
        return y > 0.0f ? y : slope * y;
    };
    const int nv = VEC ? n >> 2 : n;
#pragma unroll 2
    for (int i = blockIdx.x * 256 + threadIdx.x; i < nv; i += gridDim.x * 256) {
        if (VEC) {
            const float4 v = ld4(src, i);
            st4(dst, i, make_float4(f(v.x), f(v.y), f(v.z), f(v.w)));
        } else {
            dst[i] = f(src[i]);
        }
    }
}

// Gradient of a block output: its feature gradient (nullable) plus, when `pg`
// is set, the 2x average-pool backward of the coarser level's input gradient
// (sampling.hpp:194-219), added exactly as the separate pass would: the cell
// value g/8 once per (dx, dy, dz) that clamps onto the voxel, in order.
struct PoolSrc {
    const float *g;  // {C, od.n} or nullptr
    D3 d, od;        // fine / coarse dims
};
__device__ __forceinline__ float gz_at(const float *gz, const PoolSrc &ps, int c, int p) {
    float a = gz ? gz[(int64_t)c * ps.d.n + p] : 0.0f;
    if (ps.g) {
        const int t = p / ps.d.h, x = p - t * ps.d.h, z = t / ps.d.w, y = t - z * ps.d.w;
        const int mx = (x == ps.d.h - 1 && (ps.d.h & 1)) ? 2 : 1;
        const int my = (y == ps.d.w - 1 && (ps.d.w & 1)) ? 2 : 1;
        const int mz = (z == ps.d.l - 1 && (ps.d.l & 1)) ? 2 : 1;
        const float g =
            ps.g[(int64_t)c * ps.od.n + ((z >> 1) * ps.od.w + (y >> 1)) * ps.od.h + (x >> 1)] / 8.0f;
        for (int k = 0; k < mx * my * mz; ++k) a += g;
    }
    return a;
}
// four x-consecutive voxels from p0 (p0 % 4 == 0, h % 4 == 0 so one row and mx = 1)
__device__ __forceinline__ float4 gz_at4(const float *gz, const PoolSrc &ps, int c, int i4) {
    float4 a = gz ? ld4(gz + (int64_t)c * ps.d.n, i4) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (ps.g) {
        const int p = 4 * i4;
        const int t = p / ps.d.h, x = p - t * ps.d.h, z = t / ps.d.w, y = t - z * ps.d.w;
        const int my = (y == ps.d.w - 1 && (ps.d.w & 1)) ? 2 : 1;
        const int mz = (z == ps.d.l - 1 && (ps.d.l & 1)) ? 2 : 1;
        const float *row = ps.g + (int64_t)c * ps.od.n + ((z >> 1) * ps.od.w + (y >> 1)) * ps.od.h;
        const float g0 = row[x >> 1] / 8.0f, g1 = row[(x >> 1) + 1] / 8.0f;
        for (int k = 0; k < my * mz; ++k) {
            a.x += g0;
            a.y += g0;
            a.z += g1;
            a.w += g1;
        }
    }
    return a;
}

// backward sums per channel: gy = gz * lrelu'(y), xh = (x - mean) inv:
// part[c][blk] = {sum gy, sum gy * xh}
template <bool VEC>
__global__ void __launch_bounds__(256)
in_bwd_sum_k(const float *__restrict__ x, const float *__restrict__ gz, PoolSrc ps, int n,
             const float *__restrict__ mean, const float *__restrict__ inv,
             const float *__restrict__ g, const float *__restrict__ b, float slope,
             float *__restrict__ part) {
    const int c = blockIdx.y;
    const float mu = mean[c], iv = inv[c], gg = g[c], bb = b[c];
    const float *xs = x + (int64_t)c * n;
    float a[2] = {0.0f, 0.0f};
    auto acc = [&](float xv, float gv) {
        const float xh = (xv - mu) * iv;
        const float y = gg * xh + bb;
        const float gy = gv * (y > 0.0f ? 1.0f : slope);
        a[0] += gy;
        a[1] = fmaf(gy, xh, a[1]);
    };
    const int nv = VEC ? n >> 2 : n;
#pragma unroll 2
    for (int i = blockIdx.x * 256 + threadIdx.x; i < nv; i += gridDim.x * 256) {
        if (VEC) {
            const float4 xv = ld4(xs, i), gv = gz_at4(gz, ps, c, i);
            acc(xv.x, gv.x);
            acc(xv.y, gv.y);
            acc(xv.z, gv.z);
            acc(xv.w, gv.w);
        } else {
            acc(xs[i], gz_at(gz, ps, c, i));
        }
    }
    __shared__ float r[2];
    block_sum<2>(a, r);
    __syncthreads();
    if (threadIdx.x < 2) part[((int64_t)c * gridDim.x + blockIdx.x) * 2 + threadIdx.x] = r[threadIdx.x];
}

// sums[c] = {sum gy, sum gy xh}; gamma/beta grads accumulate
__global__ void __launch_bounds__(256)
in_bwd_final_k(const float *__restrict__ part, int nparts, float *__restrict__ sums,
               float *__restrict__ gg, float *__restrict__ gb) {
    const int c = blockIdx.x;
    float a[2] = {0.0f, 0.0f};
    for (int i = threadIdx.x; i < nparts; i += 256) {
        a[0] += part[((int64_t)c * nparts + i) * 2];
        a[1] += part[((int64_t)c * nparts + i) * 2 + 1];
    }
    __shared__ float r[2];
    block_sum<2>(a, r);
    __syncthreads();
    if (threadIdx.x == 0) {
        sums[2 * c] = r[0];
        sums[2 * c + 1] = r[1];
        if (gg) gg[c] += r[1];  // ops.hpp:204-205: gs += sum_gx, gb += sum_g
        if (gb) gb[c] += r[0];
    }
}

// gx = (gamma inv) (gy - mean(gy) - xh mean(gy xh))   (ops.hpp:206-212);
// written (not accumulated): the conv output it feeds is internal
template <bool VEC>
__global__ void __launch_bounds__(256)
in_bwd_apply_k(const float *__restrict__ x, const float *__restrict__ gz, PoolSrc ps, int n,
               const float *__restrict__ mean, const float *__restrict__ inv,
               const float *__restrict__ g, const float *__restrict__ b, float slope,
               const float *__restrict__ sums, int64_t nstat, float *__restrict__ gx) {
    // nstat: the voxel count the statistics run over (n, or the whole
    // volume's for a depth slab)
    const int c = blockIdx.y;
    const float mu = mean[c], iv = inv[c], gg = g[c], bb = b[c];
    const float k = gg * iv, mg = sums[2 * c] / (float)nstat, mgx = sums[2 * c + 1] / (float)nstat;
    const float *xs = x + (int64_t)c * n;
    float *dst = gx + (int64_t)c * n;
    auto f = [&](float xv, float gv) {
        const float xh = (xv - mu) * iv;
        const float y = gg * xh + bb;
        const float gy = gv * (y > 0.0f ? 1.0f : slope);
        return k * (gy - mg - xh * mgx);
    };
    const int nv = VEC ? n >> 2 : n;
#pragma unroll 2
    for (int i = blockIdx.x * 256 + threadIdx.x; i < nv; i += gridDim.x * 256) {
        if (VEC) {
            const float4 xv = ld4(xs, i), gv = gz_at4(gz, ps, c, i);
            st4(dst, i, make_float4(f(xv.x, gv.x), f(xv.y, gv.y), f(xv.z, gv.z), f(xv.w, gv.w)));
        } else {
            dst[i] = f(xs[i], gz_at(gz, ps, c, i));
        }
    }
}

// ---- depth-slab statistics: per-channel sums accumulated in fp64 (the
// ranks' shares are all-reduced, so their grouping must not cost accuracy).
// part[c][blk][v]; fixed order throughout.
template <int NV>
__device__ __forceinline__ void block_sum64(double (&v)[NV], double *out) {
    __shared__ double red[NV][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if (lane == 0) red[k][wid] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double a = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) a += red[threadIdx.x][w];
        out[threadIdx.x] = a;
    }
}

// NV = 1: sum x (mean == nullptr) or sum (x - mean)^2;  NV = 2: the IN
// backward's {sum gy, sum gy xh}
template <int NV>
__global__ void __launch_bounds__(256)
slab_sum64_k(const float *__restrict__ x, const float *__restrict__ gz, int n,
             const float *__restrict__ mean, const float *__restrict__ inv,
             const float *__restrict__ g, const float *__restrict__ b, float slope,
             double *__restrict__ part) {
    const int c = blockIdx.y;
    const float *xs = x + (int64_t)c * n;
    double a[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) a[k] = 0.0;
    const double mu = mean ? (double)mean[c] : 0.0;
    const float muf = mean ? mean[c] : 0.0f, iv = inv ? inv[c] : 0.0f;
    const float gg = g ? g[c] : 0.0f, bb = b ? b[c] : 0.0f;
    const float *gs = gz ? gz + (int64_t)c * n : nullptr;
    auto acc = [&](float xv, float gv) {
        if (NV == 1) {
            if (mean) {
                const double t = (double)xv - mu;
                a[0] += t * t;
            } else {
                a[0] += (double)xv;
            }
        } else {
            const float xh = (xv - muf) * iv;
            const float y = gg * xh + bb;
            const float gy = gv * (y > 0.0f ? 1.0f : slope);
            a[0] += (double)gy;
            a[NV - 1] += (double)gy * (double)xh;
        }
    };
    // float4 body (16-byte aligned channel planes when n % 4 == 0), scalar tail
    const int n4 = (n % 4 == 0) ? n / 4 : 0;
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n4; i += gridDim.x * 256) {
        const float4 v = ld4(xs, i);
        const float4 w = NV == 2 ? ld4(gs, i) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        acc(v.x, w.x);
        acc(v.y, w.y);
        acc(v.z, w.z);
        acc(v.w, w.w);
    }
    for (int i = 4 * n4 + blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256)
        acc(xs[i], NV == 2 ? gs[i] : 0.0f);
    block_sum64<NV>(a, part + ((int64_t)c * gridDim.x + blockIdx.x) * NV);
}

template <int NV>
__global__ void __launch_bounds__(256)
slab_final64_k(const double *__restrict__ part, int nparts, double *__restrict__ out) {
    const int c = blockIdx.x;
    double a[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) a[k] = 0.0;
    for (int i = threadIdx.x; i < nparts; i += 256)
#pragma unroll
        for (int k = 0; k < NV; ++k) a[k] += part[((int64_t)c * nparts + i) * NV + k];
    __shared__ double r[NV];
    block_sum64<NV>(a, r);
    __syncthreads();
    if (threadIdx.x < NV) out[c * NV + threadIdx.x] = r[threadIdx.x];
}

// ------------------------------------------------------------ avg pooling 2x
// sampling.hpp:171-191 (replicate padding for odd dims); one thread per
// output voxel, grid row per channel, 32-bit index math
__global__ void __launch_bounds__(256)
avgpool_fwd_k(const float *__restrict__ in, D3 d, D3 od, float *__restrict__ out) {
    const int c = blockIdx.y;
    const float *pl = in + (int64_t)c * d.n;
    for (int o = blockIdx.x * 256 + threadIdx.x; o < od.n; o += gridDim.x * 256) {
        const int t = o / od.h, x = o - t * od.h, z = t / od.w, y = t - z * od.w;
        const int x0 = 2 * x, x1 = min(2 * x + 1, d.h - 1);
        float s = 0.0f;
#pragma unroll
        for (int dz = 0; dz < 2; ++dz)
#pragma unroll
            for (int dy = 0; dy < 2; ++dy) {
                const int yi = min(2 * y + dy, d.w - 1), zi = min(2 * z + dz, d.l - 1);
                const float *row = pl + (zi * d.w + yi) * d.h;
                s += row[x0];
                s += row[x1];
            }
        out[(int64_t)c * od.n + o] = s / 8.0f;
    }
}

// sampling.hpp:194-219 as a gather: input (x,y,z) gets g/8 of its output
// cell once per (dx,dy,dz) that clamps onto it.  One thread per x pair (the
// pair shares its output cell).
__global__ void __launch_bounds__(256)
avgpool_bwd_k(const float *__restrict__ gout, D3 d, D3 od, float *__restrict__ gin) {
    const int c = blockIdx.y;
    const int hp = (d.h + 1) >> 1, npair = hp * d.w * d.l;
    const float *gp = gout + (int64_t)c * od.n;
    float *ip = gin + (int64_t)c * d.n;
    for (int q = blockIdx.x * 256 + threadIdx.x; q < npair; q += gridDim.x * 256) {
        const int t = q / hp, xp = q - t * hp, z = t / d.w, y = t - z * d.w;
        const int my = (y == d.w - 1 && (d.w & 1)) ? 2 : 1;
        const int mz = (z == d.l - 1 && (d.l & 1)) ? 2 : 1;
        const float g = gp[((z >> 1) * od.w + (y >> 1)) * od.h + xp] / 8.0f;
        const int x = 2 * xp, p = (z * d.w + y) * d.h + x;
        float a = ip[p];
        const int m0 = (x == d.h - 1) ? 2 * my * mz : my * mz;  // odd h: last x clamps twice
        for (int k = 0; k < m0; ++k) a += g;
        ip[p] = a;
        if (x + 1 < d.h) {
            float a1 = ip[p + 1];
            for (int k = 0; k < my * mz; ++k) a1 += g;
            ip[p + 1] = a1;
        }
    }
}

}  // namespace enc

using namespace enc;

// blocks per channel row for a plane of `items`: ~8 resident 256-thread
// blocks per SM over all C rows, at most one item per thread
static unsigned plane_blocks(int64_t items, int C) {
    const int64_t want = std::max<int64_t>(1, (148 * 8 + C - 1) / C);
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, want));
}

static unsigned grid_for(int64_t n, int per = 256) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 8));
}

// ---------------------------------------------------------------- internal
// algorithm choice (MDG_ENC_ALGO=tiled|igemm|slab forces one, benchmarking):
// TMA slab kernels (conv3t_k / conv3w_k), the implicit GEMM
// (encoder_igemm.cu), or the thread-staged slab kernels (conv3g_k /
// conv3g_wgrad_k) for volumes TMA cannot tile.
static int enc_algo() {
    static int a = [] {
        const char *e = std::getenv("MDG_ENC_ALGO");
        if (!e) return 0;
        return std::strcmp(e, "tiled") == 0   ? 1
               : std::strcmp(e, "igemm") == 0 ? 2
               : std::strcmp(e, "slab") == 0  ? 3
                                              : 0;
    }();
    return a;
}
// auto (measured at the small-preset levels, tools/bench_conv.py): the TMA
// slab kernels from ~32K voxels up when the rows are 16-B pitched; the
// implicit GEMM for smaller (deeper) levels with >= 32 output channels.
static bool use_igemm(int cout, int cin, const D3 &d) {
    if ((int64_t)cin * d.n >= (int64_t(1) << 31)) return false;
    const int a = enc_algo();
    return a == 2 || (a == 0 && cout >= 32 && (d.n < 32768 || d.h % 4 != 0));
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_fn() {
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

// 4-D map {h, w, l, C} with the conv3t_k box {40, 10, 6, CIB}; false when TMA
// cannot take the volume (row pitch not a multiple of 16 B, misaligned base)
static bool conv_map(CUtensorMap *m, const float *base, const D3 &d, int C) {
    if (enc_algo() == 3 || d.h % 4 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0 ||
        !tmap_fn())
        return false;
    const cuuint64_t dims[4] = {(cuuint64_t)d.h, (cuuint64_t)d.w, (cuuint64_t)d.l, (cuuint64_t)C};
    const cuuint64_t strides[3] = {(cuuint64_t)d.h * 4, (cuuint64_t)d.h * d.w * 4,
                                   (cuuint64_t)d.n * 4};
    const cuuint32_t box[4] = {PX, HY, HZ, CIB};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return tmap_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(base), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// conv3t_k launch: blocked weights + the TMA kernel (ACC: accumulate, no bias)
template <bool ACC>
static mdg_status conv3t_launch(const CUtensorMap &map, const float *w, int oc, int ic, bool flip,
                                const D3 &d, const float *bias, float *out, cudaStream_t st,
                                float *norm_stats = nullptr) {
    const int cin = flip ? oc : ic, cout = flip ? ic : oc;
    const int cpad = (cin + CIB - 1) / CIB * CIB, nob = (cout + OCB - 1) / OCB;
    Scratch wb;
    MDG_CUDA_TRY(wb.alloc((size_t)nob * cpad * WCH * sizeof(float), st));
    wprep_blocked_k<<<grid_for((int64_t)nob * cpad * WCH), 256, 0, st>>>(w, oc, ic, flip ? 1 : 0,
                                                                         cpad, nob, wb.as<float>());
    MDG_LAUNCHED();
    MDG_CUDA_TRY(cudaFuncSetAttribute(conv3t_k<ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)TSMEM));
    const dim3 g((d.h + TX - 1) / TX, (d.w + TY - 1) / TY, ((d.l + TV - 1) / TV) * nob);
    Scratch sp;
    const int ntx = g.x, nty = g.y, ntz = (d.l + TV - 1) / TV;
    if (norm_stats)
        MDG_CUDA_TRY(sp.alloc((size_t)cout * ntx * nty * ntz * sizeof(float2), st));
    conv3t_k<ACC><<<g, NT, TSMEM, st>>>(map, cin, d, wb.as<float>(), cpad, bias, cout, out,
                                        norm_stats ? sp.as<float2>() : nullptr);
    MDG_LAUNCHED();
    if (norm_stats) {
        in_stats_k<<<cout, 256, 0, st>>>(sp.as<float2>(), d, ntx, nty, ntz, 1e-5f, norm_stats,
                                         norm_stats + cout);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

static bool map4(CUtensorMap *m, const float *base, const D3 &d, int C, cuuint32_t bx,
                 cuuint32_t by, cuuint32_t bz, cuuint32_t bc) {
    if (enc_algo() == 3 || d.h % 4 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0 ||
        !tmap_fn())
        return false;
    const cuuint64_t dims[4] = {(cuuint64_t)d.h, (cuuint64_t)d.w, (cuuint64_t)d.l, (cuuint64_t)C};
    const cuuint64_t strides[3] = {(cuuint64_t)d.h * 4, (cuuint64_t)d.h * d.w * 4,
                                   (cuuint64_t)d.n * 4};
    const cuuint32_t box[4] = {bx, by, bz, bc};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return tmap_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(base), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA kernel gradient (conv3w_k); false if the volume does not take TMA
template <int WC, int OH>
static bool conv3w_try(const float *in, int ic, const D3 &d, const float *gout, int oc, float *gk,
                       float *gb, cudaStream_t st, mdg_status *rc) {
    using W = WT<WC, OH>;
    CUtensorMap im, gm;
    if (!map4(&im, in, d, ic, PX, HY, ZW + 2, WC) || !map4(&gm, gout, d, oc, TX, TY, ZW, OCB))
        return false;
    *rc = MDG_OK;
    const int ntx = (d.h + TX - 1) / TX, nty = (d.w + TY - 1) / TY;
    const int nob = (oc + OCB - 1) / OCB, ncc = (ic + WC - 1) / WC;
    const int base = ntx * nty * nob * ncc;
    // z split: ~4 waves of CTAs at 2-3 resident per SM, >= 8 planes each
    const int want = 148 * 3 * 4;
    int nz = std::max(1, std::min((want + base - 1) / base, (d.l + 7) / 8));
    int zper = (d.l + nz - 1) / nz;
    zper = (zper + ZW - 1) / ZW * ZW;
    nz = (d.l + zper - 1) / zper;
    const int nblk = ntx * nty * nz;
    Scratch part;
    const size_t np = (size_t)nob * ncc * nblk * OCB * WC * 27;
    cudaError_t e = part.alloc((np + (size_t)nob * nblk * OCB) * sizeof(float), st);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(conv3w_k<WC, OH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)W::SMEM);
    if (e != cudaSuccess) {
        *rc = status_from_cuda(e, "conv3w");
        return true;
    }
    float *pb = part.as<float>() + np;
    conv3w_k<WC, OH><<<dim3(ntx * nty * ncc, nz, nob), W::NTH, W::SMEM, st>>>(
        im, gm, ic, oc, d, zper, ncc, part.as<float>(), pb);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if ((e = cudaPeekAtLastError()) != cudaSuccess) {
        *rc = status_from_cuda(e, "conv3w_k");
        return true;
    }
    const int nout = oc * ic * 27 + oc;
    conv3w_sum_k<WC><<<(nout + 7) / 8, 256, 0, st>>>(part.as<float>(), pb, nblk, ncc, oc, ic, gk,
                                                     gb);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if ((e = cudaPeekAtLastError()) != cudaSuccess) *rc = status_from_cuda(e, "conv3w_sum_k");
    return true;
}

mdg_status enc_conv3_fwd(const float *in, int ic, mdg_dims3 dd, const float *w, const float *b,
                         int oc, float *out, cudaStream_t st, float *norm_stats,
                         bool *stats_done) {
    const D3 d{dd.h, dd.w, dd.l, dd.h * dd.w * dd.l};
    if (stats_done) *stats_done = false;
    // 32 / 64 output channels on a large enough grid: the tensor cores
    // (encoder_tc.cu; the normalisation statistics then run as separate passes)
    if (enc_tc_conv_ok(ic, oc, dd)) return enc_tc_conv(in, ic, dd, w, oc, 0, b, false, out, st);
    const bool ig = use_igemm(oc, ic, d);
    CUtensorMap map;
    if (!ig && conv_map(&map, in, d, ic)) {
        const bool want = norm_stats && stats_done;
        const mdg_status s =
            conv3t_launch<false>(map, w, oc, ic, false, d, b, out, st, want ? norm_stats : nullptr);
        if (s == MDG_OK && want) *stats_done = true;
        return s;
    }
    const int tile = ig ? igemm_fwd_bn(oc) : OCB;
    const int opad = (oc + tile - 1) / tile * tile;
    Scratch wt;
    MDG_CUDA_TRY(wt.alloc((size_t)ic * 27 * opad * sizeof(float), st));
    wprep_k<<<grid_for((int64_t)ic * 27 * opad), 256, 0, st>>>(w, oc, ic, 0, opad, wt.as<float>());
    MDG_LAUNCHED();
    if (ig) return igemm_conv_fwd(in, ic, dd, wt.as<float>(), opad, b, oc, false, out, st);
    const dim3 g((d.h + TX - 1) / TX, (d.w + TY - 1) / TY, ((d.l + TV - 1) / TV) * (opad / OCB));
    conv3g_k<false><<<g, NT, 0, st>>>(in, ic, d, wt.as<float>(), opad, b, oc, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status enc_conv3_bwd(const float *in, int ic, mdg_dims3 dd, const float *w, int oc,
                         const float *gout, float *gin, float *gw, float *gb, cudaStream_t st,
                         bool gin_acc) {
    const D3 d{dd.h, dd.w, dd.l, dd.h * dd.w * dd.l};
    if (gin && enc_tc_conv_ok(oc, ic, dd)) {
        // the input gradient on the tensor cores: conv of gout with the
        // flipped, transposed kernel
        if (mdg_status s = enc_tc_conv(gout, oc, dd, w, ic, 1, nullptr, gin_acc, gin, st))
            return s;
    } else if (gin) {
        const bool ig = use_igemm(ic, oc, d);
        CUtensorMap map;
        if (!ig && conv_map(&map, gout, d, oc)) {
            const mdg_status s2 =
                gin_acc ? conv3t_launch<true>(map, w, oc, ic, true, d, nullptr, gin, st)
                        : conv3t_launch<false>(map, w, oc, ic, true, d, nullptr, gin, st);
            if (s2 != MDG_OK) return s2;
        } else {
            const int tile = ig ? igemm_fwd_bn(ic) : OCB;
            const int ipad = (ic + tile - 1) / tile * tile;
            Scratch wt;
            MDG_CUDA_TRY(wt.alloc((size_t)oc * 27 * ipad * sizeof(float), st));
            wprep_k<<<grid_for((int64_t)oc * 27 * ipad), 256, 0, st>>>(w, oc, ic, 1, ipad,
                                                                       wt.as<float>());
            MDG_LAUNCHED();
            if (ig) {
                const mdg_status s =
                    igemm_conv_fwd(gout, oc, dd, wt.as<float>(), ipad, nullptr, ic, gin_acc, gin, st);
                if (s != MDG_OK) return s;
            } else {
                const dim3 g((d.h + TX - 1) / TX, (d.w + TY - 1) / TY,
                             ((d.l + TV - 1) / TV) * (ipad / OCB));
                (gin_acc ? conv3g_k<true> : conv3g_k<false>)<<<g, NT, 0, st>>>(
                    gout, oc, d, wt.as<float>(), ipad, nullptr, ic, gin);
                MDG_LAUNCHED();
            }
        }
    }
    if ((gw || gb) && use_igemm(oc, ic, d)) return igemm_conv_wgrad(in, ic, dd, gout, oc, gw, gb, st);
    if (gw || gb) {
        mdg_status rc = MDG_OK;
        static const int oh = [] {
            const char *e = std::getenv("MDG_CONV3W_OH");  // tuning override
            return e && std::atoi(e) == 1 ? 1 : 2;
        }();
        const bool done = ic == 1 ? (oh == 1 ? conv3w_try<1, 1>(in, ic, d, gout, oc, gw, gb, st, &rc)
                                             : conv3w_try<1, 2>(in, ic, d, gout, oc, gw, gb, st, &rc))
                                  : (oh == 1 ? conv3w_try<2, 1>(in, ic, d, gout, oc, gw, gb, st, &rc)
                                             : conv3w_try<2, 2>(in, ic, d, gout, oc, gw, gb, st, &rc));
        if (done) return rc;
    }
    if (gw || gb) {
        const int ntiles = ((d.h + TX - 1) / TX) * ((d.w + TY - 1) / TY) * ((d.l + TV - 1) / TV);
        const int noy = (oc + OCB - 1) / OCB, ncz = (ic + CIB - 1) / CIB;
        const int nblk = ntiles;  // one CTA per voxel block
        Scratch part;
        const size_t np = (size_t)nblk * noy * ncz * OCB * CIB * 27;
        MDG_CUDA_TRY(part.alloc((np + (size_t)nblk * noy * OCB) * sizeof(float), st));
        float *pb = part.as<float>() + np;
        const size_t smem = (size_t)(CIB * SLAB + OCB * TV * TY * TX) * sizeof(float);
        MDG_CUDA_TRY(cudaFuncSetAttribute(conv3g_wgrad_k,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        conv3g_wgrad_k<<<dim3(nblk, noy, ncz), WG_NT, smem, st>>>(in, ic, d, gout, oc,
                                                                  part.as<float>(), pb);
        MDG_LAUNCHED();
        if (nblk >= 64)
            conv3g_wgrad_tree_k<<<oc * ic * 27 + oc, 256, 0, st>>>(part.as<float>(), pb, nblk,
                                                                   noy, ncz, oc, ic, gw, gb);
        else
            conv3g_wgrad_final_k<<<(oc * ic * 27 + oc + 255) / 256, 256, 0, st>>>(
                part.as<float>(), pb, nblk, noy, ncz, oc, ic, gw, gb);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

// z = lrelu(IN(x)); mean / inv (per channel) saved for the backward
mdg_status enc_in_lrelu_fwd(const float *x, int C, int64_t n, const float *g, const float *b,
                            float slope, float *z, float *mean, float *inv, cudaStream_t st) {
    const bool vec = n % 4 == 0;
    const unsigned gx = plane_blocks(vec ? n / 4 : n, C);
    Scratch part;
    MDG_CUDA_TRY(part.alloc((size_t)C * gx * sizeof(float), st));
    auto sum = vec ? chan_sum_k<true> : chan_sum_k<false>;
    sum<<<dim3(gx, C), 256, 0, st>>>(x, (int)n, nullptr, part.as<float>());
    MDG_LAUNCHED();
    chan_final_k<<<C, 256, 0, st>>>(part.as<float>(), gx, (int)n, 0, 0.0f, mean);
    MDG_LAUNCHED();
    sum<<<dim3(gx, C), 256, 0, st>>>(x, (int)n, mean, part.as<float>());
    MDG_LAUNCHED();
    chan_final_k<<<C, 256, 0, st>>>(part.as<float>(), gx, (int)n, 1, 1e-5f, inv);
    MDG_LAUNCHED();
    (vec ? in_apply_k<true> : in_apply_k<false>)<<<dim3(gx, C), 256, 0, st>>>(x, (int)n, mean, inv,
                                                                            g, b, slope, z);
    MDG_LAUNCHED();
    return MDG_OK;
}

// z = lrelu(IN(x)) with mean / inv already known (fused into the conv)
mdg_status enc_in_lrelu_apply(const float *x, int C, int64_t n, const float *g, const float *b,
                              float slope, float *z, const float *mean, const float *inv,
                              cudaStream_t st) {
    const bool vec = n % 4 == 0;
    const unsigned gx = plane_blocks(vec ? n / 4 : n, C);
    (vec ? in_apply_k<true> : in_apply_k<false>)<<<dim3(gx, C), 256, 0, st>>>(x, (int)n, mean, inv,
                                                                            g, b, slope, z);
    MDG_LAUNCHED();
    return MDG_OK;
}

// gx = d/dx of lrelu(IN(x)) applied to gz (written); gamma/beta grads accumulate
mdg_status enc_in_lrelu_bwd(const float *x, const float *gz, const float *pg, mdg_dims3 fd,
                            int C, int64_t n, const float *g, const float *b, float slope,
                            const float *mean, const float *inv, float *gx, float *gg,
                            float *gbeta, cudaStream_t st) {
    const D3 d{fd.h, fd.w, fd.l, fd.h * fd.w * fd.l};
    const int oh = (fd.h + 1) / 2, ow = (fd.w + 1) / 2, ol = (fd.l + 1) / 2;
    const PoolSrc ps{pg, d, D3{oh, ow, ol, oh * ow * ol}};
    const bool vec = n % 4 == 0 && fd.h % 4 == 0;
    const unsigned nb = plane_blocks(vec ? n / 4 : n, C);
    Scratch part;
    MDG_CUDA_TRY(part.alloc(((size_t)C * nb * 2 + 2 * C) * sizeof(float), st));
    float *sums = part.as<float>() + (size_t)C * nb * 2;
    (vec ? in_bwd_sum_k<true> : in_bwd_sum_k<false>)<<<dim3(nb, C), 256, 0, st>>>(
        x, gz, ps, (int)n, mean, inv, g, b, slope, part.as<float>());
    MDG_LAUNCHED();
    in_bwd_final_k<<<C, 256, 0, st>>>(part.as<float>(), nb, sums, gg, gbeta);
    MDG_LAUNCHED();
    (vec ? in_bwd_apply_k<true> : in_bwd_apply_k<false>)<<<dim3(nb, C), 256, 0, st>>>(
        x, gz, ps, (int)n, mean, inv, g, b, slope, sums, n, gx);
    MDG_LAUNCHED();
    return MDG_OK;
}

// ---- depth-slab instance norm: the same kernels with the statistics'
// sums exposed, so a caller can all-reduce them between the passes
// sums[c] = sum x (mean == nullptr) or sum (x - mean[c])^2 over this slab (fp64)
mdg_status enc_in_slab_sums(const float *x, int C, int64_t n, const float *mean, double *sums,
                            cudaStream_t st) {
    const unsigned gx = plane_blocks(n % 4 == 0 ? n / 4 : n, C);
    Scratch part;
    MDG_CUDA_TRY(part.alloc((size_t)C * gx * sizeof(double), st));
    slab_sum64_k<1><<<dim3(gx, C), 256, 0, st>>>(x, nullptr, (int)n, mean, nullptr, nullptr,
                                                nullptr, 0.0f, part.as<double>());
    MDG_LAUNCHED();
    slab_final64_k<1><<<C, 256, 0, st>>>(part.as<double>(), gx, sums);
    MDG_LAUNCHED();
    return MDG_OK;
}

// sums[2c..2c+1] = {sum gy, sum gy xh} over this slab (gy = gz lrelu'(y); fp64)
mdg_status enc_in_slab_bwd_sums(const float *x, const float *gz, int C, int64_t n,
                                const float *g, const float *b, float slope, const float *mean,
                                const float *inv, double *sums, cudaStream_t st) {
    const unsigned nb = plane_blocks(n % 4 == 0 ? n / 4 : n, C);
    Scratch part;
    MDG_CUDA_TRY(part.alloc((size_t)C * nb * 2 * sizeof(double), st));
    slab_sum64_k<2><<<dim3(nb, C), 256, 0, st>>>(x, gz, (int)n, mean, inv, g, b, slope,
                                                part.as<double>());
    MDG_LAUNCHED();
    slab_final64_k<2><<<C, 256, 0, st>>>(part.as<double>(), nb, sums);
    MDG_LAUNCHED();
    return MDG_OK;
}

// gx (written) from the all-reduced sums over nstat voxels
mdg_status enc_in_slab_bwd_apply(const float *x, const float *gz, int C, int64_t n,
                                 const float *g, const float *b, float slope, const float *mean,
                                 const float *inv, const float *sums, int64_t nstat, float *gx,
                                 cudaStream_t st) {
    // no pooled gradient: only d.n (gz's channel stride) is read
    const PoolSrc ps{nullptr, D3{1, 1, 1, (int)n}, D3{1, 1, 1, 1}};
    const bool vec = n % 4 == 0;
    const unsigned nb = plane_blocks(vec ? n / 4 : n, C);
    (vec ? in_bwd_apply_k<true> : in_bwd_apply_k<false>)<<<dim3(nb, C), 256, 0, st>>>(
        x, gz, ps, (int)n, mean, inv, g, b, slope, sums, nstat, gx);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status enc_avgpool_fwd(const float *in, int C, mdg_dims3 dd, float *out, cudaStream_t st) {
    const D3 d{dd.h, dd.w, dd.l, dd.h * dd.w * dd.l};
    const int oh = (dd.h + 1) / 2, ow = (dd.w + 1) / 2, ol = (dd.l + 1) / 2;
    const D3 od{oh, ow, ol, oh * ow * ol};
    avgpool_fwd_k<<<dim3(plane_blocks(od.n, C), C), 256, 0, st>>>(in, d, od, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status enc_avgpool_bwd(const float *gout, int C, mdg_dims3 dd, float *gin, cudaStream_t st) {
    const D3 d{dd.h, dd.w, dd.l, dd.h * dd.w * dd.l};
    const int oh = (dd.h + 1) / 2, ow = (dd.w + 1) / 2, ol = (dd.l + 1) / 2;
    const D3 od{oh, ow, ol, oh * ow * ol};
    avgpool_bwd_k<<<dim3(plane_blocks((int64_t)((dd.h + 1) / 2) * dd.w * dd.l, C), C), 256, 0, st>>>(
        gout, d, od, gin);
    MDG_LAUNCHED();
    return MDG_OK;
}

}  // namespace mdg
