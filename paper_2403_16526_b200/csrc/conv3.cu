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
#include "mdg_common.cuh"

namespace mdg {

constexpr int kCB = 256;
constexpr int kChunkPerThread = 8;

__device__ __forceinline__ void xyz3(int64_t p, int h, int w, int &x, int &y, int &z) {
    x = (int)(p % h);
    const int64_t t = p / h;
    y = (int)(t % w);
    z = (int)(t / w);
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
