// Experiment: the warp backward's gin scatter into a channel-last (voxel-major,
// C = 8) accumulator with 16-byte vector reductions (red.global.add.v4.f32):
// 8 corners x 2 vector REDs per voxel instead of 8 x 8 scalar ones, then one
// pass adds the channel-last sums into the planar gin.  Weights and terms as
// sampling.hpp:103-118 ((g*wx)*wy)*wz.
#include <cuda_runtime.h>
#include <cstdint>

struct Ax { int i0, i1; float f; };
__device__ __forceinline__ Ax resolve(float x, int dim) {
    Ax a;
    const float hi = (float)(dim - 1);
    const float xc = x < 0.0f ? 0.0f : (x > hi ? hi : x);
    int i0 = (int)floorf(xc);
    if (i0 > dim - 2) i0 = dim - 2;
    a.i0 = i0; a.i1 = i0 + 1; a.f = __fsub_rn(xc, (float)i0);
    return a;
}
__device__ __forceinline__ void red4(float *a, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 sc4(float4 g, float w) {
    return make_float4(__fmul_rn(g.x, w), __fmul_rn(g.y, w), __fmul_rn(g.z, w), __fmul_rn(g.w, w));
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB)
scatter_cl_k(const float *__restrict__ field, const float *__restrict__ gout, int h, int w, int l,
             float *__restrict__ gcl) {
    const int64_t n = (int64_t)h * w * l;
    const int p = blockIdx.x * 256 + threadIdx.x;
    if (p >= n) return;
    const int t = p / h, x = p - t * h, z = t / w, y = t - z * w;
    const Ax ax = resolve(__fadd_rn((float)x, __ldg(field + p)), h);
    const Ax ay = resolve(__fadd_rn((float)y, __ldg(field + n + p)), w);
    const Ax az = resolve(__fadd_rn((float)z, __ldg(field + 2 * n + p)), l);
    float4 g0, g1;
    g0.x = __ldg(gout + p); g0.y = __ldg(gout + n + p); g0.z = __ldg(gout + 2 * n + p);
    g0.w = __ldg(gout + 3 * n + p); g1.x = __ldg(gout + 4 * n + p); g1.y = __ldg(gout + 5 * n + p);
    g1.z = __ldg(gout + 6 * n + p); g1.w = __ldg(gout + 7 * n + p);
    const float wx[2] = {__fsub_rn(1.0f, ax.f), ax.f}, wy[2] = {__fsub_rn(1.0f, ay.f), ay.f};
    const float wz[2] = {__fsub_rn(1.0f, az.f), az.f};
    const int xs[2] = {ax.i0, ax.i1}, ys[2] = {ay.i0, ay.i1}, zs[2] = {az.i0, az.i1};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
        const int64_t q = ((int64_t)zs[dz] * w + ys[dy]) * h + xs[dx];
        // ((g*wx)*wy)*wz per channel, as the reference
        const float4 a = sc4(sc4(sc4(g0, wx[dx]), wy[dy]), wz[dz]);
        const float4 b = sc4(sc4(sc4(g1, wx[dx]), wy[dy]), wz[dz]);
        red4(gcl + 8 * q, a);
        red4(gcl + 8 * q + 4, b);
    }
}

// gin[c][p] += gcl[p][c]
__global__ void add_cl_k(const float *__restrict__ gcl, int64_t n, float *__restrict__ gin) {
    const int64_t p = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (p >= n) return;
    const float4 a = reinterpret_cast<const float4 *>(gcl)[2 * p];
    const float4 b = reinterpret_cast<const float4 *>(gcl)[2 * p + 1];
    gin[p] += a.x; gin[n + p] += a.y; gin[2 * n + p] += a.z; gin[3 * n + p] += a.w;
    gin[4 * n + p] += b.x; gin[5 * n + p] += b.y; gin[6 * n + p] += b.z; gin[7 * n + p] += b.w;
}

extern "C" int scatter_cl(const float *field, const float *gout, int h, int w, int l, float *gcl,
                          float *gin, int minb, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (int64_t)h * w * l;
    cudaMemsetAsync(gcl, 0, n * 8 * sizeof(float), st);
    const unsigned g = (unsigned)((n + 255) / 256);
    if (minb == 4) scatter_cl_k<4><<<g, 256, 0, st>>>(field, gout, h, w, l, gcl);
    else if (minb == 6) scatter_cl_k<6><<<g, 256, 0, st>>>(field, gout, h, w, l, gcl);
    else scatter_cl_k<8><<<g, 256, 0, st>>>(field, gout, h, w, l, gcl);
    add_cl_k<<<g, 256, 0, st>>>(gcl, n, gin);
    return (int)cudaPeekAtLastError();
}
extern "C" int scatter_only(const float *field, const float *gout, int h, int w, int l, float *gcl,
                            void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (int64_t)h * w * l;
    scatter_cl_k<6><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(field, gout, h, w, l, gcl);
    return (int)cudaPeekAtLastError();
}
