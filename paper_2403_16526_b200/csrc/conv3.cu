// conv3.cu — zero-padded 3x3x3 convolution (correlation) on sm_100a: the
// RegHead fusion of the 3S sub-flow channels into one 3-channel field
// (reghead.hpp:42-47 -> ops.hpp:137-158).
//
// fwd and the input gradient are gathers whose per-element term order equals
// the reference's slab loops (ops.hpp:27-37, 58-99), so both are bit-identical
// to the CPU reference.  The kernel/bias gradients are full-volume reductions:
// per-CTA partials over fixed voxel chunks, then a fixed-order tree — the
// result is deterministic (run to run) and within fp32 reduction tolerance of
// the reference's sequential sums.
#include <algorithm>

#include "mdg_common.cuh"

namespace mdg {

constexpr int kCB = 256;
constexpr int kChunkPerThread = 8;

__device__ __forceinline__ void xyz3(int64_t p, int h, int w, int &x, int &y, int &z) {
    const int p32 = (int)p;  // n < 2^31 (dims_ok): 32-bit div/mod
    const int t = p32 / h;
    x = p32 - t * h;
    z = t / w;
    y = t - z * w;
}

// ops.hpp:58-74
__global__ void __launch_bounds__(kCB)
conv3_fwd_k(const float *__restrict__ in, int ic, int h, int w, int l,
            const float *__restrict__ k, const float *__restrict__ bias, int oc,
            float *__restrict__ out) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kCB + threadIdx.x;
    if (p >= n) return;
    int x, y, z;
    xyz3(p, h, w, x, y, z);
    const int64_t hw = (int64_t)h * w;
    for (int co = 0; co < oc; ++co) {
        float acc = bias ? __ldg(bias + co) : 0.0f;
        for (int ci = 0; ci < ic; ++ci) {
            const float *kk = k + ((int64_t)co * ic + ci) * 27;
            const float *src = in + (int64_t)ci * n + p;
#pragma unroll
            for (int t = 0; t < 27; ++t) {
                const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
                const float kv = __ldg(kk + t);
                if (kv == 0.0f) continue;
                if (x + dx < 0 || x + dx >= h || y + dy < 0 || y + dy >= w || z + dz < 0 ||
                    z + dz >= l)
                    continue;
                acc = add_(acc, mul_(kv, __ldg(src + dx + dy * (int64_t)h + dz * hw)));
            }
        }
        out[(int64_t)co * n + p] = acc;
    }
}

// ops.hpp:95-96 (gin += kv * gout shifted back), order (co, tap)
__global__ void __launch_bounds__(kCB)
conv3_bwd_in_k(int ic, int h, int w, int l, const float *__restrict__ k, int oc,
               const float *__restrict__ gout, float *__restrict__ gin) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kCB + threadIdx.x;
    if (p >= n) return;
    int x, y, z;
    xyz3(p, h, w, x, y, z);
    const int64_t hw = (int64_t)h * w;
    for (int ci = 0; ci < ic; ++ci) {
        float acc = gin[(int64_t)ci * n + p];
        for (int co = 0; co < oc; ++co) {
            const float *kk = k + ((int64_t)co * ic + ci) * 27;
            const float *g = gout + (int64_t)co * n + p;
#pragma unroll
            for (int t = 0; t < 27; ++t) {
                const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
                const float kv = __ldg(kk + t);
                if (kv == 0.0f) continue;
                if (x - dx < 0 || x - dx >= h || y - dy < 0 || y - dy >= w || z - dz < 0 ||
                    z - dz >= l)
                    continue;
                acc = add_(acc, mul_(kv, __ldg(g - dx - dy * (int64_t)h - dz * hw)));
            }
        }
        gin[(int64_t)ci * n + p] = acc;
    }
}

// per-CTA partial sums of gk[co,ci,:] (27 taps) and, for ci == 0, gbias[co]
// over a fixed chunk of kCB*kChunkPerThread voxels (ops.hpp:80-85, 93-94)
__global__ void __launch_bounds__(kCB)
conv3_bwd_w_parts_k(const float *__restrict__ in, int ic, int h, int w, int l,
                    const float *__restrict__ gout, int oc, float *__restrict__ part) {
    const int64_t n = (int64_t)h * w * l;
    const int pair = blockIdx.y;  // co * ic + ci
    const int co = pair / ic, ci = pair % ic;
    const int64_t hw = (int64_t)h * w;
    float acc[28];
#pragma unroll
    for (int t = 0; t < 28; ++t) acc[t] = 0.0f;
    const int64_t base = (int64_t)blockIdx.x * kCB * kChunkPerThread;
    for (int it = 0; it < kChunkPerThread; ++it) {
        const int64_t p = base + (int64_t)it * kCB + threadIdx.x;
        if (p >= n) break;
        int x, y, z;
        xyz3(p, h, w, x, y, z);
        const float g = __ldg(gout + (int64_t)co * n + p);
        acc[27] += g;
        const float *src = in + (int64_t)ci * n + p;
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
            if (x + dx < 0 || x + dx >= h || y + dy < 0 || y + dy >= w || z + dz < 0 ||
                z + dz >= l)
                continue;
            acc[t] = fmaf(g, __ldg(src + dx + dy * (int64_t)h + dz * hw), acc[t]);
        }
    }
    __shared__ float red[kCB / 32][28];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int t = 0; t < 28; ++t) {
        float v = acc[t];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) red[wid][t] = v;
    }
    __syncthreads();
    if (threadIdx.x < 28) {
        float v = 0.0f;
#pragma unroll
        for (int i = 0; i < kCB / 32; ++i) v += red[i][threadIdx.x];
        part[((int64_t)pair * gridDim.x + blockIdx.x) * 28 + threadIdx.x] = v;
    }
}

__global__ void __launch_bounds__(kCB)
conv3_bwd_w_final_k(const float *__restrict__ part, int nparts, int ic,
                    float *__restrict__ gk, float *__restrict__ gbias) {
    const int pair = blockIdx.y, t = blockIdx.x;  // t in [0, 28)
    if (t == 27 && (pair % ic != 0 || !gbias)) return;
    if (t < 27 && !gk) return;
    float v = 0.0f;
    for (int i = threadIdx.x; i < nparts; i += kCB) v += part[((int64_t)pair * nparts + i) * 28 + t];
    __shared__ float sm[kCB];
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int m = kCB / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) sm[threadIdx.x] += sm[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (t < 27) gk[(int64_t)pair * 27 + t] += sm[0];
        else gbias[pair / ic] += sm[0];
    }
}

// ------------------------------------------------------------ tiled (oc == 3)
// The RegHead shape (3S -> 3).  A CTA of 32x8 threads covers a 32x8x4 block:
// each thread owns one (x, y) column of kV = 4 consecutive z voxels, so every
// weight read from shared memory feeds kV voxels and every staged tap value
// feeds all three output channels.  Input planes z0-1 .. z0+kV of a chunk of
// channels are staged with a one-voxel zero halo, so taps need no bounds
// checks.  Each output keeps the reference's term order (bias, then
// channel-major, taps dz/dy/dx) with products and sums rounded separately and
// zero weights skipped (ops.hpp:69): fwd and gin are bit-identical to the CPU
// reference (an out-of-range tap adds kv*0 = +-0, leaving the sum unchanged).
constexpr int kTX = 32, kTY = 8, kV = 4;
constexpr int kHX = kTX + 2, kHY = kTY + 2, kHZ = kV + 2;
constexpr int kPlaneXY = kHY * kHX;
constexpr int kSlab = kHZ * kPlaneXY;  // one channel: kV+2 z planes with halo
constexpr int kChunk = 2;             // channels staged per pass

// Staging of nch channel slabs: every element the thread copies is first
// loaded into registers (all loads in flight together), then stored, so a
// stage costs about one global-load latency instead of one per element.
// Rows are kHX wide; lanes run along x, so the index decomposition and the
// y/z bounds test are per row.  nch <= kMaxStageCh.
constexpr int kStageRows = kHZ * kHY;  // per channel

template <int MAXCH>
__device__ __forceinline__ void stage_slab(float *dst, const float *__restrict__ src, int nch,
                                           int h, int w, int l, int x0, int y0, int z0) {
    constexpr int kRowIters = (MAXCH * kStageRows + 7) / 8;  // per warp (8 warps)
    const int64_t n = (int64_t)h * w * l;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int rows = nch * kStageRows;
    const int gx0 = x0 - 1 + lane, gx1 = x0 - 1 + lane + 32;
    const bool okx0 = gx0 >= 0 && gx0 < h, okx1 = lane + 32 < kHX && gx1 < h;
    float v0[kRowIters], v1[kRowIters];
#pragma unroll
    for (int it = 0; it < kRowIters; ++it) {
        const int r = wid + 8 * it;
        v0[it] = 0.0f;
        v1[it] = 0.0f;
        if (r < rows) {
            const int c = r / kStageRows, rr = r - c * kStageRows;
            const int dz = rr / kHY, yy = rr - dz * kHY;
            const int gy = y0 - 1 + yy, gz = z0 - 1 + dz;
            if (gy >= 0 && gy < w && gz >= 0 && gz < l) {
                const float *srow = src + (int64_t)c * n + ((int64_t)gz * w + gy) * h;
                if (okx0) v0[it] = __ldg(srow + gx0);
                if (okx1) v1[it] = __ldg(srow + gx1);
            }
        }
    }
#pragma unroll
    for (int it = 0; it < kRowIters; ++it) {
        const int r = wid + 8 * it;
        if (r < rows) {
            dst[r * kHX + lane] = v0[it];
            if (lane + 32 < kHX) dst[r * kHX + lane + 32] = v1[it];
        }
    }
}

template <int OC>
__global__ void __launch_bounds__(kTX *kTY, 2)
conv3_fwd_tiled_k(const float *__restrict__ in, int ic, int h, int w, int l,
                  const float *__restrict__ k, const float *__restrict__ bias,
                  float *__restrict__ out) {
    extern __shared__ float sm[];
    float *kw = sm;                   // [OC][ic][27]
    float *slab = sm + OC * ic * 27;  // [kChunk][kHZ][kHY][kHX]
    for (int i = threadIdx.x; i < OC * ic * 27; i += blockDim.x) kw[i] = k[i];
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY, z0 = blockIdx.z * kV;
    float acc[kV][OC];
#pragma unroll
    for (int co = 0; co < OC; ++co) {
        const float b0 = bias ? __ldg(bias + co) : 0.0f;
#pragma unroll
        for (int v = 0; v < kV; ++v) acc[v][co] = b0;
    }
    for (int c0 = 0; c0 < ic; c0 += kChunk) {
        const int nch = min(kChunk, ic - c0);
        __syncthreads();
        stage_slab<kChunk>(slab, in + (int64_t)c0 * h * w * l, nch, h, w, l, x0, y0, z0);
        __syncthreads();
        for (int cc = 0; cc < nch; ++cc) {
            const float *tp = slab + cc * kSlab + ty * kHX + tx;
            const float *kc = kw + (c0 + cc) * 27;
#pragma unroll
            for (int t = 0; t < 27; ++t) {
                const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
                float xv[kV];
#pragma unroll
                for (int v = 0; v < kV; ++v) xv[v] = tp[((v + dz) * kHY + dy) * kHX + dx];
#pragma unroll
                for (int co = 0; co < OC; ++co) {
                    const float kv = kc[co * ic * 27 + t];
                    if (kv == 0.0f) continue;  // ops.hpp:69 (uniform)
#pragma unroll
                    for (int v = 0; v < kV; ++v) acc[v][co] = add_(acc[v][co], mul_(kv, xv[v]));
                }
            }
        }
    }
    const int x = x0 + tx, y = y0 + ty;
    if (x >= h || y >= w) return;
    const int64_t n = (int64_t)h * w * l;
#pragma unroll
    for (int v = 0; v < kV; ++v) {
        if (z0 + v >= l) break;
        const int64_t p = ((int64_t)(z0 + v) * w + y) * h + x;
#pragma unroll
        for (int co = 0; co < OC; ++co) out[co * n + p] = acc[v][co];
    }
}

// gin[ci] += sum_co sum_t k[co,ci,t] gout[co](p - off(t)), order (co, t)
// (ops.hpp:94-96).  gout planes are staged once; tap t of voxel v reads slab
// position (v + 2 - dz, ty + 2 - dy, tx + 2 - dx).
template <int OC>
__global__ void __launch_bounds__(kTX *kTY)
conv3_bwd_in_tiled_k(int ic, int h, int w, int l, const float *__restrict__ k,
                     const float *__restrict__ gout, float *__restrict__ gin) {
    extern __shared__ float sm[];
    float *kw = sm;
    float *slab = sm + OC * ic * 27;  // [OC][kHZ][kHY][kHX] of gout
    for (int i = threadIdx.x; i < OC * ic * 27; i += blockDim.x) kw[i] = k[i];
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY, z0 = blockIdx.z * kV;
    stage_slab<OC>(slab, gout, OC, h, w, l, x0, y0, z0);
    __syncthreads();
    const int x = x0 + tx, y = y0 + ty;
    if (x >= h || y >= w) return;
    const int64_t n = (int64_t)h * w * l;
    const int nv = min(kV, l - z0);
    const int64_t p0 = ((int64_t)z0 * w + y) * h + x, hw = (int64_t)h * w;
    const float *tp = slab + ty * kHX + tx;
    for (int ci = 0; ci < ic; ++ci) {
        float acc[kV];
#pragma unroll
        for (int v = 0; v < kV; ++v) acc[v] = v < nv ? gin[(int64_t)ci * n + p0 + v * hw] : 0.0f;
#pragma unroll
        for (int co = 0; co < OC; ++co) {
            const float *kk = kw + (co * ic + ci) * 27;
            const float *gp = tp + co * kSlab;
#pragma unroll
            for (int t = 0; t < 27; ++t) {
                const float kv = kk[t];
                if (kv == 0.0f) continue;
                const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
                for (int v = 0; v < kV; ++v)
                    acc[v] = add_(acc[v], mul_(kv, gp[((v + 2 - dz) * kHY + (2 - dy)) * kHX + (2 - dx)]));
            }
        }
#pragma unroll
        for (int v = 0; v < kV; ++v)
            if (v < nv) gin[(int64_t)ci * n + p0 + v * hw] = acc[v];
    }
}

// kernel / bias gradients: blockIdx.y = input channel ci; a persistent grid
// walks the 32x8x4 blocks, staging channel ci's slab (kV+2 planes with halo)
// in shared memory; each thread holds gout of its kV voxels for all OC output
// channels and accumulates acc[co][t] += gout[co](p) * in[ci](p + off(t)) in
// registers (every staged tap value feeds OC accumulators), + the bias sums on
// ci == 0; then a fixed-order block reduction -> per-CTA partials ->
// fixed-order final sum (deterministic).
template <int OC>
__global__ void __launch_bounds__(kTX *kTY, 2)
conv3_bwd_w_tiled_k(const float *__restrict__ in, int ic, int h, int w, int l,
                    const float *__restrict__ gout, float *__restrict__ part) {
    __shared__ float slab[2][kSlab];
    __shared__ float red[kTX * kTY / 32];
    const int ci = blockIdx.y;
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    const int ntx = (h + kTX - 1) / kTX, nty = (w + kTY - 1) / kTY, ntz = (l + kV - 1) / kV;
    const int ntiles = ntx * nty * ntz;
    const int64_t n = (int64_t)h * w * l, hw = (int64_t)h * w;
    float acc[OC][27], accb[OC];
#pragma unroll
    for (int co = 0; co < OC; ++co) {
        accb[co] = 0.0f;
#pragma unroll
        for (int t = 0; t < 27; ++t) acc[co][t] = 0.0f;
    }
    const float *src = in + (int64_t)ci * n;
    // double-buffered staging: tile i+1's slab streams in (cp.async, zero
    // fill outside the volume) while tile i is accumulated
    auto stage_async = [&](float *dst, int ti) {
        const int bx = ti % ntx, by = (ti / ntx) % nty, bz = ti / (ntx * nty);
        const int x0 = bx * kTX, y0 = by * kTY, z0 = bz * kV;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int r = wid; r < kStageRows; r += 8) {
            const int dz = r / kHY, yy = r - dz * kHY;
            const int gy = y0 - 1 + yy, gz = z0 - 1 + dz;
            const bool rowok = gy >= 0 && gy < w && gz >= 0 && gz < l;
            const float *srow = src + ((int64_t)(rowok ? gz : 0) * w + (rowok ? gy : 0)) * h;
            for (int xx = lane; xx < kHX; xx += 32) {
                const int gx = x0 - 1 + xx;
                const bool ok = rowok && gx >= 0 && gx < h;
                const unsigned d = (unsigned)__cvta_generic_to_shared(dst + r * kHX + xx);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d),
                             "l"(ok ? srow + gx : src), "r"(ok ? 4 : 0));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    int buf = 0;
    if ((int)blockIdx.x < ntiles) stage_async(slab[0], blockIdx.x);
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const int tn = ti + gridDim.x;
        if (tn < ntiles) {
            stage_async(slab[buf ^ 1], tn);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        const int bx = ti % ntx, by = (ti / ntx) % nty, bz = ti / (ntx * nty);
        const int x0 = bx * kTX, y0 = by * kTY, z0 = bz * kV;
        const int x = x0 + tx, y = y0 + ty;
        const bool inxy = x < h && y < w;
        const int64_t p0 = ((int64_t)z0 * w + y) * h + x;
        float g[kV][OC];
#pragma unroll
        for (int v = 0; v < kV; ++v) {
            const bool ok = inxy && z0 + v < l;
#pragma unroll
            for (int co = 0; co < OC; ++co) {
                g[v][co] = ok ? __ldg(gout + co * n + p0 + v * hw) : 0.0f;
                accb[co] += g[v][co];
            }
        }
        const float *tp = slab[buf] + ty * kHX + tx;
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                const float xv = tp[((v + dz) * kHY + dy) * kHX + dx];
#pragma unroll
                for (int co = 0; co < OC; ++co) acc[co][t] = fmaf(g[v][co], xv, acc[co][t]);
            }
        }
        __syncthreads();  // buffer `buf` is refilled two tiles later
        buf ^= 1;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *dst = part + ((int64_t)ci * gridDim.x + blockIdx.x) * (OC * 28);
    auto reduce = [&](float v, int slot) {
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) red[wid] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            float sum = 0.0f;
#pragma unroll
            for (int i = 0; i < kTX * kTY / 32; ++i) sum += red[i];
            dst[slot] = sum;
        }
        __syncthreads();
    };
#pragma unroll
    for (int co = 0; co < OC; ++co) {
#pragma unroll
        for (int t = 0; t < 27; ++t) reduce(acc[co][t], co * 28 + t);
        reduce(accb[co], co * 28 + 27);
    }
}

// gk[co,ci,t] += sum over CTAs; gbias[co] += (ci == 0 partials only)
template <int OC>
__global__ void __launch_bounds__(256)
conv3_bwd_w_tiled_final_k(const float *__restrict__ part, int nparts, int ic,
                          float *__restrict__ gk, float *__restrict__ gbias) {
    const int ci = blockIdx.y, slot = blockIdx.x;  // slot = co*28 + t
    const int co = slot / 28, t = slot % 28;
    if (t == 27 && (ci != 0 || !gbias)) return;
    if (t < 27 && !gk) return;
    float v = 0.0f;
    for (int i = threadIdx.x; i < nparts; i += 256)
        v += part[((int64_t)ci * nparts + i) * (OC * 28) + slot];
    __shared__ float s[256];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int m = 128; m > 0; m >>= 1) {
        if (threadIdx.x < m) s[threadIdx.x] += s[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (t < 27) gk[((int64_t)co * ic + ci) * 27 + t] += s[0];
        else gbias[co] += s[0];
    }
}

}  // namespace mdg

using namespace mdg;

extern "C" {

mdg_status mdg_conv3_fwd(const float *in, int ic, mdg_dims3 d, const float *k,
                         const float *bias, int oc, float *out, void *stream) {
    MDG_REQUIRE(ic >= 1 && oc >= 1, "conv3: channel counts must be >= 1");
    MDG_REQUIRE(dims_ok(d), "conv3: invalid dims " + dims_str(d));
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(in && k && out, "conv3: null pointer");
    if (oc == 3 && ic <= 64) {  // RegHead: tiled shared-memory path
        const size_t smem = (size_t)(3 * ic * 27 + kChunk * kSlab) * sizeof(float);
        const dim3 g((d.h + kTX - 1) / kTX, (d.w + kTY - 1) / kTY, (d.l + kV - 1) / kV);
        conv3_fwd_tiled_k<3><<<g, kTX * kTY, smem, S_(stream)>>>(in, ic, d.h, d.w, d.l, k, bias,
                                                                 out);
        MDG_LAUNCHED();
        return MDG_OK;
    }
    conv3_fwd_k<<<grid1d(n, kCB), kCB, 0, S_(stream)>>>(in, ic, d.h, d.w, d.l, k, bias, oc, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_conv3_bwd(const float *in, int ic, mdg_dims3 d, const float *k, int oc,
                         const float *gout, float *gin, float *gk, float *gbias, void *stream) {
    MDG_REQUIRE(ic >= 1 && oc >= 1, "conv3: channel counts must be >= 1");
    MDG_REQUIRE(dims_ok(d), "conv3: invalid dims " + dims_str(d));
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(in && k && gout, "conv3: null pointer");
    cudaStream_t st = S_(stream);
    if (oc == 3 && ic <= 64) {  // RegHead: tiled shared-memory path
        const dim3 g((d.h + kTX - 1) / kTX, (d.w + kTY - 1) / kTY, (d.l + kV - 1) / kV);
        if (gin) {
            const size_t smem = (size_t)(3 * ic * 27 + 3 * kSlab) * sizeof(float);
            conv3_bwd_in_tiled_k<3><<<g, kTX * kTY, smem, st>>>(ic, d.h, d.w, d.l, k, gout, gin);
            MDG_LAUNCHED();
        }
        if (gk || gbias) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int64_t ntiles = (int64_t)g.x * g.y * g.z;
            const int gx = (int)std::max<int64_t>(
                1, std::min<int64_t>(ntiles, ((int64_t)sms * 2 + ic - 1) / ic));
            Scratch part;
            MDG_CUDA_TRY(part.alloc((size_t)ic * gx * 3 * 28 * sizeof(float), st));
            conv3_bwd_w_tiled_k<3><<<dim3(gx, ic), kTX * kTY, 0, st>>>(in, ic, d.h, d.w, d.l, gout,
                                                                      part.as<float>());
            MDG_LAUNCHED();
            conv3_bwd_w_tiled_final_k<3><<<dim3(3 * 28, ic), 256, 0, st>>>(part.as<float>(), gx,
                                                                           ic, gk, gbias);
            MDG_LAUNCHED();
        }
        return MDG_OK;
    }
    if (gin) {
        conv3_bwd_in_k<<<grid1d(n, kCB), kCB, 0, st>>>(ic, d.h, d.w, d.l, k, oc, gout, gin);
        MDG_LAUNCHED();
    }
    if (gk || gbias) {
        const int nparts = (int)((n + kCB * kChunkPerThread - 1) / (kCB * kChunkPerThread));
        Scratch part;
        MDG_CUDA_TRY(part.alloc((size_t)oc * ic * nparts * 28 * sizeof(float), st));
        conv3_bwd_w_parts_k<<<dim3(nparts, oc * ic), kCB, 0, st>>>(in, ic, d.h, d.w, d.l, gout,
                                                                    oc, part.as<float>());
        MDG_LAUNCHED();
        conv3_bwd_w_final_k<<<dim3(28, oc * ic), kCB, 0, st>>>(part.as<float>(), nparts, ic, gk,
                                                               gbias);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

}  // extern "C"
