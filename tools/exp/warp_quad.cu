// Experiment: like warp_ypair.cu with each thread owning a 2 x 2 (y, z) quad
// of voxels: y-pairs merge their shared y rows, then the two pairs merge
// their shared z rows — 9 corner rows per quad instead of 16 when the
// field is locally smooth.  gin only, C = 8 (dev experiment).
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
__device__ __forceinline__ float m_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ void red_if(float *a, float v, bool p) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q red.global.add.f32 [%0], %1;\n}\n"
                 ::"l"(a), "f"(v), "r"((int)p) : "memory");
}
__device__ __forceinline__ void xmerge(int r, bool ok, bool &in, bool &out) {
    const int lane = threadIdx.x & 31;
    const int key = ok ? r : -2 - lane;
    const int up = __shfl_up_sync(0xffffffffu, ok ? r + 1 : -1, 1);
    in = lane > 0 && ok && up == key;
    out = __shfl_down_sync(0xffffffffu, (int)in, 1) != 0 && lane < 31;
}
__device__ __forceinline__ void emit(float *plane, int r, bool ok, float t0, float t1, bool in,
                                     bool out) {
    const float nx = __shfl_up_sync(0xffffffffu, t1, 1);
    red_if(plane + r, in ? t0 + nx : t0, ok);
    red_if(plane + r + 1, t1, ok && !out);
}

struct Vox {
    Ax ax, ay, az;
    bool ok;
    int p;
};
__device__ __forceinline__ Vox vox(const float *field, int64_t n, int h, int w, int l, int x, int y,
                                   int z, bool ok) {
    Vox v;
    v.ok = ok;
    v.p = ok ? (z * w + y) * h + x : 0;
    v.ax = resolve(__fadd_rn((float)x, __ldg(field + v.p)), h);
    v.ay = resolve(__fadd_rn((float)y, __ldg(field + n + v.p)), w);
    v.az = resolve(__fadd_rn((float)z, __ldg(field + 2 * n + v.p)), l);
    return v;
}
__device__ __forceinline__ int row(const Vox &v, int jy, int jz, int h, int hw) {
    return (jz ? v.az.i1 : v.az.i0) * hw + (jy ? v.ay.i1 : v.ay.i0) * h + v.ax.i0;
}
// the four (x0, x1) terms of voxel v's row (jy, jz) for upstream g
__device__ __forceinline__ void terms(const Vox &v, float g, int jy, int jz, float &t0, float &t1) {
    const float wy = jy ? v.ay.f : __fsub_rn(1.0f, v.ay.f);
    const float wz = jz ? v.az.f : __fsub_rn(1.0f, v.az.f);
    t0 = m_(m_(m_(g, __fsub_rn(1.0f, v.ax.f)), wy), wz);
    t1 = m_(m_(m_(g, v.ax.f), wy), wz);
}

template <int C>
__global__ void __launch_bounds__(256, 2)
quad_k(const float *__restrict__ field, const float *__restrict__ gout, int h, int w, int l,
       float *__restrict__ gin) {
    const int64_t n = (int64_t)h * w * l;
    const int wp = (w + 1) / 2, lp = (l + 1) / 2;
    const int64_t nq = (int64_t)h * wp * lp;
    const int64_t q0 = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const bool live = q0 < nq;
    const int q = live ? (int)q0 : 0;
    const int t = q / h, x = q - t * h, zq = t / wp, yq = t - zq * wp;
    const int y0 = 2 * yq, z0 = 2 * zq;
    const int hw = h * w;
    // voxels: V[dy + 2 dz]
    Vox V[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        V[k] = vox(field, n, h, w, l, x, y0 + (k & 1), z0 + (k >> 1),
                   live && y0 + (k & 1) < w && z0 + (k >> 1) < l);
    // y-pair merges (A,B) and (C,D); z merge of the pairs
    const bool my0 = V[1].ok && row(V[0], 1, 0, h, hw) == row(V[1], 0, 0, h, hw) &&
                     row(V[0], 1, 1, h, hw) == row(V[1], 0, 1, h, hw);
    const bool my1 = V[3].ok && row(V[2], 1, 0, h, hw) == row(V[3], 0, 0, h, hw) &&
                     row(V[2], 1, 1, h, hw) == row(V[3], 0, 1, h, hw);
    const bool mz = my0 && my1 && V[2].ok && row(V[0], 0, 1, h, hw) == row(V[2], 0, 0, h, hw) &&
                    row(V[0], 1, 1, h, hw) == row(V[2], 1, 0, h, hw) &&
                    row(V[1], 1, 1, h, hw) == row(V[3], 1, 0, h, hw);
    // 16 warp-uniform slots: slot (k, jy, jz) = voxel k's row (jy, jz), with
    // merged rows carried by the lower voxel / lower pair and disabled on
    // the other
    int rs[16];
    bool oks[16], in[16], out[16];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int jy = j & 1, jz = j >> 1;
            bool ok = V[k].ok;
            // a y-merged pair: the upper voxel's y0 rows go to the lower voxel's y1 rows
            if ((k & 1) && jy == 0 && ((k >> 1) ? my1 : my0)) ok = false;
            // z-merged pairs: the upper pair's z0 rows go to the lower pair's z1 rows
            if ((k >> 1) && jz == 0 && mz) ok = false;
            rs[4 * k + j] = row(V[k], jy, jz, h, hw);
            oks[4 * k + j] = ok;
        }
#pragma unroll
    for (int s = 0; s < 16; ++s) xmerge(rs[s], oks[s], in[s], out[s]);
#pragma unroll 1
    for (int c = 0; c < C; ++c) {
        float g[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) g[k] = V[k].ok ? __ldg(gout + (int64_t)c * n + V[k].p) : 0.0f;
        float T0[16], T1[16];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < 4; ++j) terms(V[k], g[k], j & 1, j >> 1, T0[4 * k + j], T1[4 * k + j]);
        // fold merged rows into their carriers (y first, then z)
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
            const bool my = pr ? my1 : my0;
            const int lo = 2 * pr, hi = 2 * pr + 1;  // voxel indices
            if (my) {
#pragma unroll
                for (int jz = 0; jz < 2; ++jz) {  // hi's (y0, jz) -> lo's (y1, jz)
                    T0[4 * lo + 1 + 2 * jz] += T0[4 * hi + 0 + 2 * jz];
                    T1[4 * lo + 1 + 2 * jz] += T1[4 * hi + 0 + 2 * jz];
                }
            }
        }
        if (mz) {
            // upper pair's z0 rows -> lower pair's z1 rows: C (y0,z0)->A (y0,z1),
            // C (y1,z0) [= D (y0,z0) merged] -> A (y1,z1), D (y1,z0) -> B (y1,z1)
            T0[0 + 2] += T0[8 + 0]; T1[0 + 2] += T1[8 + 0];
            T0[0 + 3] += T0[8 + 1]; T1[0 + 3] += T1[8 + 1];
            T0[4 + 3] += T0[12 + 1]; T1[4 + 3] += T1[12 + 1];
        }
        float *pl = gin + (int64_t)c * n;
#pragma unroll
        for (int s = 0; s < 16; ++s) emit(pl, rs[s], oks[s], T0[s], T1[s], in[s], out[s]);
    }
}

extern "C" int quad_gin(const float *field, const float *gout, int h, int w, int l, float *gin,
                        void *stream) {
    const int64_t nq = (int64_t)h * ((w + 1) / 2) * ((l + 1) / 2);
    quad_k<8><<<(unsigned)((nq + 255) / 256), 256, 0, (cudaStream_t)stream>>>(field, gout, h, w, l,
                                                                            gin);
    return (int)cudaPeekAtLastError();
}
