// Experiment: the warp backward's gin scatter with each thread owning a
// y-pair of voxels (x, y) and (x, y+1).  For a smooth field the pair's corner
// rows overlap (A's y1 rows are B's y0 rows): those two rows are merged in
// registers, 6 corner rows per pair instead of 8, i.e. 25 % fewer fp32
// reductions reach the L2; the warp-level x-merge of lane t's x1 term into
// lane t+1's x0 term applies on top.  gin only, C = 8 (dev experiment).
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
// lane t absorbs lane t-1's x1 term when that lands on its own x0 target
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

template <int C, int MINB>
__global__ void __launch_bounds__(256, MINB)
ypair_k(const float *__restrict__ field, const float *__restrict__ gout, int h, int w, int l,
        float *__restrict__ gin) {
    const int64_t n = (int64_t)h * w * l;
    const int wp = (w + 1) / 2;
    const int64_t np = (int64_t)h * wp * l;
    const int64_t q0 = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const bool live = q0 < np;
    const int q = live ? (int)q0 : 0;
    const int t = q / h, x = q - t * h, z = t / wp, yp = t - z * wp;
    const int yA = 2 * yp, yB = yA + 1;
    const bool okA = live, okB = live && yB < w;
    const int pA = (z * w + yA) * h + x, pB = okB ? pA + h : pA;
    const Ax axA = resolve(__fadd_rn((float)x, __ldg(field + pA)), h);
    const Ax ayA = resolve(__fadd_rn((float)yA, __ldg(field + n + pA)), w);
    const Ax azA = resolve(__fadd_rn((float)z, __ldg(field + 2 * n + pA)), l);
    const Ax axB = resolve(__fadd_rn((float)x, __ldg(field + pB)), h);
    const Ax ayB = resolve(__fadd_rn((float)yB, __ldg(field + n + pB)), w);
    const Ax azB = resolve(__fadd_rn((float)z, __ldg(field + 2 * n + pB)), l);
    const int hw = h * w;
    // row starts (x0 included) of the 8 corner rows
    const int rA[4] = {azA.i0 * hw + ayA.i0 * h + axA.i0, azA.i0 * hw + ayA.i1 * h + axA.i0,
                       azA.i1 * hw + ayA.i0 * h + axA.i0, azA.i1 * hw + ayA.i1 * h + axA.i0};
    const int rB[4] = {azB.i0 * hw + ayB.i0 * h + axB.i0, azB.i0 * hw + ayB.i1 * h + axB.i0,
                       azB.i1 * hw + ayB.i0 * h + axB.i0, azB.i1 * hw + ayB.i1 * h + axB.i0};
    // merge: A's y1 rows (1, 3) are B's y0 rows (0, 2)
    const bool mrg = okB && rA[1] == rB[0] && rA[3] == rB[2];
    // 6 warp-uniform slots: A y0z0, A y1z0 (+B y0z0), B y1z0, A y0z1, A y1z1 (+B y0z1),
    // B y1z1; plus 2 slots for B's y0 rows when not merged
    const int rs[8] = {rA[0], rA[1], rB[1], rA[2], rA[3], rB[3], rB[0], rB[2]};
    const bool oks[8] = {okA, okA, okB, okA, okA, okB, okB && !mrg, okB && !mrg};
    bool in[8], out[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) xmerge(rs[s], oks[s], in[s], out[s]);
    const float wxA0 = __fsub_rn(1.0f, axA.f), wxA1 = axA.f, wyA0 = __fsub_rn(1.0f, ayA.f),
                wyA1 = ayA.f, wzA0 = __fsub_rn(1.0f, azA.f), wzA1 = azA.f;
    const float wxB0 = __fsub_rn(1.0f, axB.f), wxB1 = axB.f, wyB0 = __fsub_rn(1.0f, ayB.f),
                wyB1 = ayB.f, wzB0 = __fsub_rn(1.0f, azB.f), wzB1 = azB.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const float gA = __ldg(gout + (int64_t)c * n + pA);
        const float gB = okB ? __ldg(gout + (int64_t)c * n + pB) : 0.0f;
        float *pl = gin + (int64_t)c * n;
        const float a0 = m_(gA, wxA0), a1 = m_(gA, wxA1);
        const float b0 = m_(gB, wxB0), b1 = m_(gB, wxB1);
        const float a00 = m_(a0, wyA0), a10 = m_(a1, wyA0), a01 = m_(a0, wyA1), a11 = m_(a1, wyA1);
        const float b00 = m_(b0, wyB0), b10 = m_(b1, wyB0), b01 = m_(b0, wyB1), b11 = m_(b1, wyB1);
        // slot terms (x0, x1)
        const float tA_y0z0_0 = m_(a00, wzA0), tA_y0z0_1 = m_(a10, wzA0);
        const float tA_y1z0_0 = m_(a01, wzA0), tA_y1z0_1 = m_(a11, wzA0);
        const float tA_y0z1_0 = m_(a00, wzA1), tA_y0z1_1 = m_(a10, wzA1);
        const float tA_y1z1_0 = m_(a01, wzA1), tA_y1z1_1 = m_(a11, wzA1);
        const float tB_y0z0_0 = m_(b00, wzB0), tB_y0z0_1 = m_(b10, wzB0);
        const float tB_y1z0_0 = m_(b01, wzB0), tB_y1z0_1 = m_(b11, wzB0);
        const float tB_y0z1_0 = m_(b00, wzB1), tB_y0z1_1 = m_(b10, wzB1);
        const float tB_y1z1_0 = m_(b01, wzB1), tB_y1z1_1 = m_(b11, wzB1);
        emit(pl, rs[0], oks[0], tA_y0z0_0, tA_y0z0_1, in[0], out[0]);
        emit(pl, rs[1], oks[1], mrg ? tA_y1z0_0 + tB_y0z0_0 : tA_y1z0_0,
             mrg ? tA_y1z0_1 + tB_y0z0_1 : tA_y1z0_1, in[1], out[1]);
        emit(pl, rs[2], oks[2], tB_y1z0_0, tB_y1z0_1, in[2], out[2]);
        emit(pl, rs[3], oks[3], tA_y0z1_0, tA_y0z1_1, in[3], out[3]);
        emit(pl, rs[4], oks[4], mrg ? tA_y1z1_0 + tB_y0z1_0 : tA_y1z1_0,
             mrg ? tA_y1z1_1 + tB_y0z1_1 : tA_y1z1_1, in[4], out[4]);
        emit(pl, rs[5], oks[5], tB_y1z1_0, tB_y1z1_1, in[5], out[5]);
        emit(pl, rs[6], oks[6], tB_y0z0_0, tB_y0z0_1, in[6], out[6]);
        emit(pl, rs[7], oks[7], tB_y0z1_0, tB_y0z1_1, in[7], out[7]);
    }
}

extern "C" int ypair_gin_b(const float *field, const float *gout, int h, int w, int l, float *gin,
                           int minb, void *stream) {
    const int64_t np = (int64_t)h * ((w + 1) / 2) * l;
    const unsigned g = (unsigned)((np + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    if (minb == 2) ypair_k<8, 2><<<g, 256, 0, st>>>(field, gout, h, w, l, gin);
    else if (minb == 4) ypair_k<8, 4><<<g, 256, 0, st>>>(field, gout, h, w, l, gin);
    else ypair_k<8, 3><<<g, 256, 0, st>>>(field, gout, h, w, l, gin);
    return (int)cudaPeekAtLastError();
}
extern "C" int ypair_gin(const float *field, const float *gout, int h, int w, int l, float *gin,
                         void *stream) {
    return ypair_gin_b(field, gout, h, w, l, gin, 3, stream);
}
