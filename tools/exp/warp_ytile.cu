// Experiment: the warp backward's gin scatter with a 32 (x) x 8 (y) voxel
// tile per CTA (one warp per y row, one voxel per thread, so the gathers keep
// their one-voxel overlap) and a cross-warp y merge through shared memory:
// warp w's y1 corner rows usually coincide with warp w+1's y0 rows (smooth
// field); those terms are handed down and added before the x merge, so ~44 %
// fewer fp32 reductions reach the L2.  gin only or gin + gfield, C = 8.
#include <cuda_runtime.h>
#include <cstdint>

struct Ax { int i0; float f; bool live; };
__device__ __forceinline__ Ax resolve(float x, int dim) {
    Ax a;
    const float hi = (float)(dim - 1);
    const float xc = x < 0.0f ? 0.0f : (x > hi ? hi : x);
    int i0 = (int)floorf(xc);
    if (i0 > dim - 2) i0 = dim - 2;
    a.i0 = i0; a.f = __fsub_rn(xc, (float)i0); a.live = x > 0.0f && x < hi;
    return a;
}
__device__ __forceinline__ float m_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float a_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ void redf(float *a, float v, bool p) {
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
__device__ __forceinline__ void emit(float *plane, int r, bool ok, float t0, float t1, bool in, bool out) {
    const float nx = __shfl_up_sync(0xffffffffu, t1, 1);
    redf(plane + r, in ? t0 + nx : t0, ok);
    redf(plane + r + 1, t1, ok && !out);
}

template <int C, bool YM, bool GF>
__global__ void __launch_bounds__(256, 3)
ytile_k(const float *__restrict__ in, const float *__restrict__ field,
        const float *__restrict__ gout, int h, int w, int l, float *__restrict__ gin,
        float *__restrict__ gfield) {
    __shared__ int keys[8][32][2];    // y0 rows (z0, z1) of each voxel, -1: none
    __shared__ float hand[8][32][8];  // y1-row terms handed to the next warp (2 channels)
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    const int ntx = (h + 31) / 32, nty = (w + 7) / 8;
    const int b = blockIdx.x, tx = b % ntx, ty = (b / ntx) % nty, z = b / (ntx * nty);
    const int x = tx * 32 + lane, y = ty * 8 + wy;
    const bool ok = x < h && y < w;
    const int64_t n = (int64_t)h * w * l;
    const int p = ok ? (z * w + y) * h + x : 0;
    const Ax ax = resolve(__fadd_rn((float)x, __ldg(field + p)), h);
    const Ax ay = resolve(__fadd_rn((float)y, __ldg(field + n + p)), w);
    const Ax az = resolve(__fadd_rn((float)z, __ldg(field + 2 * n + p)), l);
    const int hw = h * w;
    const int r00 = az.i0 * hw + ay.i0 * h + ax.i0, r10 = r00 + h;
    const int r01 = r00 + hw, r11 = r01 + h;
    bool dn0 = false, dn1 = false, up0 = false, up1 = false;
    if (YM) {
        keys[wy][lane][0] = ok ? r00 : -1;
        keys[wy][lane][1] = ok ? r01 : -1;
        __syncthreads();
        if (ok && wy < 7) {
            dn0 = keys[wy + 1][lane][0] == r10;
            dn1 = keys[wy + 1][lane][1] == r11;
        }
        if (ok && wy > 0) {  // the warp above hands its y1 rows down
            up0 = keys[wy - 1][lane][0] != -1 && keys[wy - 1][lane][0] + h == r00;
            up1 = keys[wy - 1][lane][1] != -1 && keys[wy - 1][lane][1] + h == r01;
        }
    }
    bool in_[4], out_[4];
    xmerge(r00, ok, in_[0], out_[0]);
    xmerge(r10, ok && !dn0, in_[1], out_[1]);
    xmerge(r01, ok, in_[2], out_[2]);
    xmerge(r11, ok && !dn1, in_[3], out_[3]);
    const float wx0 = __fsub_rn(1.0f, ax.f), wx1 = ax.f, wy0 = __fsub_rn(1.0f, ay.f), wy1 = ay.f,
                wz0 = __fsub_rn(1.0f, az.f), wz1 = az.f;
    float gv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) gv[c] = ok ? __ldg(gout + (int64_t)c * n + p) : 0.0f;
    float gx = 0.0f, gy = 0.0f, gz = 0.0f;
    if (GF) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const float *a = in + (int64_t)c * n;
            const float v000 = __ldg(a + r00), v100 = __ldg(a + r00 + 1), v010 = __ldg(a + r10),
                        v110 = __ldg(a + r10 + 1), v001 = __ldg(a + r01), v101 = __ldg(a + r01 + 1),
                        v011 = __ldg(a + r11), v111 = __ldg(a + r11 + 1);
            const float cgx = ax.live ? a_(m_(a_(m_(__fsub_rn(v100, v000), wy0), m_(__fsub_rn(v110, v010), wy1)), wz0),
                                           m_(a_(m_(__fsub_rn(v101, v001), wy0), m_(__fsub_rn(v111, v011), wy1)), wz1)) : 0.0f;
            const float cgy = ay.live ? a_(m_(a_(m_(__fsub_rn(v010, v000), wx0), m_(__fsub_rn(v110, v100), wx1)), wz0),
                                           m_(a_(m_(__fsub_rn(v011, v001), wx0), m_(__fsub_rn(v111, v101), wx1)), wz1)) : 0.0f;
            const float cgz = az.live ? a_(m_(a_(m_(__fsub_rn(v001, v000), wx0), m_(__fsub_rn(v101, v100), wx1)), wy0),
                                           m_(a_(m_(__fsub_rn(v011, v010), wx0), m_(__fsub_rn(v111, v110), wx1)), wy1)) : 0.0f;
            gx = a_(gx, m_(gv[c], cgx));
            gy = a_(gy, m_(gv[c], cgy));
            gz = a_(gz, m_(gv[c], cgz));
        }
    }
#pragma unroll
    for (int c = 0; c < C; c += 2) {
        float t[2][8];  // per channel: y0z0 (x0,x1), y1z0, y0z1, y1z1
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const float g = gv[c + u];
            const float g0 = m_(g, wx0), g1 = m_(g, wx1);
            const float a00 = m_(g0, wy0), a10 = m_(g1, wy0), a01 = m_(g0, wy1), a11 = m_(g1, wy1);
            t[u][0] = m_(a00, wz0); t[u][1] = m_(a10, wz0);
            t[u][2] = m_(a01, wz0); t[u][3] = m_(a11, wz0);
            t[u][4] = m_(a00, wz1); t[u][5] = m_(a10, wz1);
            t[u][6] = m_(a01, wz1); t[u][7] = m_(a11, wz1);
        }
        if (YM) {
            // hand the y1-row terms down, add the ones handed from above
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                hand[wy][lane][4 * u + 0] = dn0 ? t[u][2] : 0.0f;
                hand[wy][lane][4 * u + 1] = dn0 ? t[u][3] : 0.0f;
                hand[wy][lane][4 * u + 2] = dn1 ? t[u][6] : 0.0f;
                hand[wy][lane][4 * u + 3] = dn1 ? t[u][7] : 0.0f;
            }
            __syncthreads();
            if (wy > 0) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (up0) {
                        t[u][0] += hand[wy - 1][lane][4 * u + 0];
                        t[u][1] += hand[wy - 1][lane][4 * u + 1];
                    }
                    if (up1) {
                        t[u][4] += hand[wy - 1][lane][4 * u + 2];
                        t[u][5] += hand[wy - 1][lane][4 * u + 3];
                    }
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            float *pl = gin + (int64_t)(c + u) * n;
            emit(pl, r00, ok, t[u][0], t[u][1], in_[0], out_[0]);
            emit(pl, r10, ok && !dn0, t[u][2], t[u][3], in_[1], out_[1]);
            emit(pl, r01, ok, t[u][4], t[u][5], in_[2], out_[2]);
            emit(pl, r11, ok && !dn1, t[u][6], t[u][7], in_[3], out_[3]);
        }
    }
    if (GF && ok) {
        gfield[p] += gx;
        gfield[n + p] += gy;
        gfield[2 * n + p] += gz;
    }
}

extern "C" int ytile_bwd(const float *in, const float *field, const float *gout, int h, int w,
                         int l, float *gin, float *gfield, int ym, int gf, void *s) {
    const unsigned g = (unsigned)(((h + 31) / 32) * ((w + 7) / 8) * l);
    cudaStream_t st = (cudaStream_t)s;
    if (ym && gf) ytile_k<8, true, true><<<g, 256, 0, st>>>(in, field, gout, h, w, l, gin, gfield);
    else if (ym) ytile_k<8, true, false><<<g, 256, 0, st>>>(in, field, gout, h, w, l, gin, gfield);
    else if (gf) ytile_k<8, false, true><<<g, 256, 0, st>>>(in, field, gout, h, w, l, gin, gfield);
    else ytile_k<8, false, false><<<g, 256, 0, st>>>(in, field, gout, h, w, l, gin, gfield);
    return (int)cudaPeekAtLastError();
}
