// sampling.cu — trilinear warp, flow composition, 2x field upsampling and
// scaling-and-squaring on sm_100a.
//
// Forward kernels gather: one thread per output voxel, the 8 corners of every
// channel read through L1.  The coordinate is the IEEE sum float(x) + phi and
// every lerp keeps the reference's multiply/multiply/add rounding
// (sampling.hpp:53-68, no FMA contraction), so warp / compose / upsample
// forwards are bit-identical to the CPU reference.
//
// Backward: the field gradient is a gather (bit-identical: the reference's
// per-channel order is kept); the image gradient is the reference's 8-corner
// scatter (sampling.hpp:103-118) done with native fp32 RED.ADD — every term is
// bit-identical, only the summation order at a shared corner varies.  The
// upsample backward is a pure gather over the <=5 candidate fine voxels per
// axis (no atomics).
#include <functional>
#include <cstdlib>

#include "mdg_common.cuh"

namespace mdg {

constexpr int kSB = 256;
constexpr int kGatherReach = kGinGatherReach;

struct Corners {
    Ax ax, ay, az;
    int o00, o10, o01, o11;  // plane offsets of the (y,z) corner rows (n < 2^31)
};

__device__ __forceinline__ Corners corners_at(float cx, float cy, float cz, int h, int w, int l) {
    Corners c;
    c.ax = resolve_axis(cx, h);
    c.ay = resolve_axis(cy, w);
    c.az = resolve_axis(cz, l);
    const int sy = h, sz = h * w;
    c.o00 = c.az.i0 * sz + c.ay.i0 * sy;
    c.o10 = c.az.i0 * sz + c.ay.i1 * sy;
    c.o01 = c.az.i1 * sz + c.ay.i0 * sy;
    c.o11 = c.az.i1 * sz + c.ay.i1 * sy;
    return c;
}

// Buffer geometry of one warp launch.  Whole volume: channel strides n, no
// offsets, the window [0, l).  Depth slab (mdg_warp_*_slab): `in`/`gin` hold
// only the planes [zlo, zhi) (channel stride csi; io = zlo*h*w is subtracted
// from every corner offset) and field/out/gout/gfield only the launch's own
// voxels (channel stride csv; voxel p is element p - vo); a voxel whose
// corners leave [zlo, zhi) touches nothing and raises *err.
struct WarpWin {
    int64_t csi, csv, vo;
    int zlo, zhi, io;
    unsigned *err;
};
inline WarpWin whole_win(int64_t n, int l) { return WarpWin{n, n, 0, 0, l, 0, nullptr}; }
// the window test; on success the corner offsets become window-relative
__device__ __forceinline__ bool in_window(Corners &c, const WarpWin &win) {
    if (c.az.i0 < win.zlo || c.az.i1 >= win.zhi) {
        if (win.err) atomicOr(win.err, 1u);
        return false;
    }
    c.o00 -= win.io;
    c.o10 -= win.io;
    c.o01 -= win.io;
    c.o11 -= win.io;
    return true;
}

// sampling.hpp:53-68
__device__ __forceinline__ float sample(const float *__restrict__ pl, const Corners &c) {
    const int x0 = c.ax.i0, dx = c.ax.i1 - c.ax.i0;  // dx = 0 on a collapsed axis
    const float fx = c.ax.f;
    const float *r00 = pl + (c.o00 + x0), *r10 = pl + (c.o10 + x0);
    const float *r01 = pl + (c.o01 + x0), *r11 = pl + (c.o11 + x0);
    const float c00 = lerp_(__ldg(r00), __ldg(r00 + dx), fx);
    const float c10 = lerp_(__ldg(r10), __ldg(r10 + dx), fx);
    const float c01 = lerp_(__ldg(r01), __ldg(r01 + dx), fx);
    const float c11 = lerp_(__ldg(r11), __ldg(r11 + dx), fx);
    const float c0 = lerp_(c00, c10, c.ay.f);
    const float c1 = lerp_(c01, c11, c.ay.f);
    return lerp_(c0, c1, c.az.f);
}

// sampling.hpp:73-99 (zero on dead axes)
__device__ __forceinline__ void sample_grad(const float *__restrict__ pl, const Corners &c,
                                            float g[3]) {
    const int x0 = c.ax.i0, dx = c.ax.i1 - c.ax.i0;
    const float *r00 = pl + (c.o00 + x0), *r10 = pl + (c.o10 + x0);
    const float *r01 = pl + (c.o01 + x0), *r11 = pl + (c.o11 + x0);
    const float v000 = __ldg(r00), v100 = __ldg(r00 + dx);
    const float v010 = __ldg(r10), v110 = __ldg(r10 + dx);
    const float v001 = __ldg(r01), v101 = __ldg(r01 + dx);
    const float v011 = __ldg(r11), v111 = __ldg(r11 + dx);
    const float fx = c.ax.f, fy = c.ay.f, fz = c.az.f;
    const float gx = sub_(1.0f, fx), gy = sub_(1.0f, fy), gz = sub_(1.0f, fz);
    g[0] = g[1] = g[2] = 0.0f;
    if (c.ax.live)
        g[0] = add_(mul_(add_(mul_(sub_(v100, v000), gy), mul_(sub_(v110, v010), fy)), gz),
                    mul_(add_(mul_(sub_(v101, v001), gy), mul_(sub_(v111, v011), fy)), fz));
    if (c.ay.live)
        g[1] = add_(mul_(add_(mul_(sub_(v010, v000), gx), mul_(sub_(v110, v100), fx)), gz),
                    mul_(add_(mul_(sub_(v011, v001), gx), mul_(sub_(v111, v101), fx)), fz));
    if (c.az.live)
        g[2] = add_(mul_(add_(mul_(sub_(v001, v000), gx), mul_(sub_(v101, v100), fx)), gy),
                    mul_(add_(mul_(sub_(v011, v010), gx), mul_(sub_(v111, v110), fx)), fy));
}

// sampling.hpp:103-118 with native fp32 reductions
__device__ __forceinline__ void scatter(float *__restrict__ gp, const Corners &c, float g) {
    const int x0 = c.ax.i0, dx = c.ax.i1 - c.ax.i0;
    const float wx0 = sub_(1.0f, c.ax.f), wx1 = c.ax.f;
    const float wy0 = sub_(1.0f, c.ay.f), wy1 = c.ay.f;
    const float wz0 = sub_(1.0f, c.az.f), wz1 = c.az.f;
    float *r00 = gp + (c.o00 + x0), *r10 = gp + (c.o10 + x0);
    float *r01 = gp + (c.o01 + x0), *r11 = gp + (c.o11 + x0);
    atomicAdd(r00, mul_(mul_(mul_(g, wx0), wy0), wz0));
    atomicAdd(r00 + dx, mul_(mul_(mul_(g, wx1), wy0), wz0));
    atomicAdd(r10, mul_(mul_(mul_(g, wx0), wy1), wz0));
    atomicAdd(r10 + dx, mul_(mul_(mul_(g, wx1), wy1), wz0));
    atomicAdd(r01, mul_(mul_(mul_(g, wx0), wy0), wz1));
    atomicAdd(r01 + dx, mul_(mul_(mul_(g, wx1), wy0), wz1));
    atomicAdd(r11, mul_(mul_(mul_(g, wx0), wy1), wz1));
    atomicAdd(r11 + dx, mul_(mul_(mul_(g, wx1), wy1), wz1));
}

// voxel counts are < 2^31 (dims_ok), so the decomposition runs in 32-bit
// integer arithmetic: a 64-bit div/mod pair costs ~10x more instructions
__device__ __forceinline__ void xyz_of(int64_t p, int h, int w, int &x, int &y, int &z) {
    const int p32 = (int)p;
    const int t = p32 / h;
    x = p32 - t * h;
    z = t / w;
    y = t - z * w;
}

// the 8 corner values of one channel plane (sampling.hpp:79-86 naming)
struct Oct {
    float v000, v100, v010, v110, v001, v101, v011, v111;
};
__device__ __forceinline__ Oct load_oct(const float *__restrict__ pl, const Corners &c) {
    const int x0 = c.ax.i0, dx = c.ax.i1 - c.ax.i0;
    const float *r00 = pl + (c.o00 + x0), *r10 = pl + (c.o10 + x0);
    const float *r01 = pl + (c.o01 + x0), *r11 = pl + (c.o11 + x0);
    return Oct{__ldg(r00), __ldg(r00 + dx), __ldg(r10), __ldg(r10 + dx),
               __ldg(r01), __ldg(r01 + dx), __ldg(r11), __ldg(r11 + dx)};
}
// sampling.hpp:53-68 on loaded corners
__device__ __forceinline__ float lerp_oct(const Oct &o, const Corners &c) {
    const float fx = c.ax.f;
    const float c00 = lerp_(o.v000, o.v100, fx), c10 = lerp_(o.v010, o.v110, fx);
    const float c01 = lerp_(o.v001, o.v101, fx), c11 = lerp_(o.v011, o.v111, fx);
    return lerp_(lerp_(c00, c10, c.ay.f), lerp_(c01, c11, c.ay.f), c.az.f);
}
// sampling.hpp:73-99 on loaded corners
__device__ __forceinline__ void grad_oct(const Oct &o, const Corners &c, float g[3]) {
    const float fx = c.ax.f, fy = c.ay.f, fz = c.az.f;
    const float gx = sub_(1.0f, fx), gy = sub_(1.0f, fy), gz = sub_(1.0f, fz);
    g[0] = g[1] = g[2] = 0.0f;
    if (c.ax.live)
        g[0] = add_(mul_(add_(mul_(sub_(o.v100, o.v000), gy), mul_(sub_(o.v110, o.v010), fy)), gz),
                    mul_(add_(mul_(sub_(o.v101, o.v001), gy), mul_(sub_(o.v111, o.v011), fy)), fz));
    if (c.ay.live)
        g[1] = add_(mul_(add_(mul_(sub_(o.v010, o.v000), gx), mul_(sub_(o.v110, o.v100), fx)), gz),
                    mul_(add_(mul_(sub_(o.v011, o.v001), gx), mul_(sub_(o.v111, o.v101), fx)), fz));
    if (c.az.live)
        g[2] = add_(mul_(add_(mul_(sub_(o.v001, o.v000), gx), mul_(sub_(o.v101, o.v100), fx)), gy),
                    mul_(add_(mul_(sub_(o.v011, o.v010), gx), mul_(sub_(o.v111, o.v110), fx)), fy));
}

// --------------------------------------------------------------- warp fwd
// sampling.hpp:123-135.  CT > 0: channel count known at compile time, all
// 8*CT corner loads issued before any interpolation (memory-level
// parallelism); CT == 0: runtime channel loop.
template <int CT, bool SLAB = false>
__global__ void __launch_bounds__(kSB, CT > 0 ? 8 : 1)
warp_fwd_k(const float *__restrict__ in, int C, int h, int w, int l,
           const float *__restrict__ field, float *__restrict__ out, int64_t pb, int64_t pe,
           WarpWin win) {
    const int64_t p = pb + (int64_t)blockIdx.x * kSB + threadIdx.x;  // voxels [pb, pe)
    if (p >= pe) return;
    int x, y, z;
    xyz_of(p, h, w, x, y, z);
    // in / out channel strides, voxel p's field/out element (SLAB: WarpWin)
    const int64_t n = SLAB ? win.csi : (int64_t)h * w * l, m = SLAB ? win.csv : n;
    const int64_t vi = SLAB ? p - win.vo : p;
    Corners c = corners_at(add_((float)x, __ldg(field + vi)), add_((float)y, __ldg(field + m + vi)),
                           add_((float)z, __ldg(field + 2 * m + vi)), h, w, l);
    if (SLAB && !in_window(c, win)) return;
    if (CT > 0) {
        // 32-bit element offsets of the 4 corner rows (x0 corner; x1 = +1)
        const int r00 = c.o00 + c.ax.i0, r10 = c.o10 + c.ax.i0;
        const int r01 = c.o01 + c.ax.i0, r11 = c.o11 + c.ax.i0;
        const float fx = c.ax.f, fy = c.ay.f, fz = c.az.f;
        const float2 FX = make_float2(fx, fx), GX = make_float2(sub_(1.0f, fx), sub_(1.0f, fx));
        const float2 FY = make_float2(fy, fy), GY = make_float2(sub_(1.0f, fy), sub_(1.0f, fy));
        const float2 FZ = make_float2(fz, fz), GZ = make_float2(sub_(1.0f, fz), sub_(1.0f, fz));
        // lerp a*(1-f) + b*f on channel pairs, each lane rounded like the
        // reference's scalar code (sampling.hpp:61-67)
        // (scalar _rn per lane: ptxas fuses packed mul+add into FFMA2 even for
        // mul.rn.f32x2 / add.rn.f32x2, which would break bit-exactness)
        auto lerp2 = [](float2 a, float2 b, float2 g, float2 f) {
            return make_float2(add_(mul_(a.x, g.x), mul_(b.x, f.x)),
                               add_(mul_(a.y, g.y), mul_(b.y, f.y)));
        };
        // two channel pairs' corner loads (32 values) in flight at once
        constexpr int G = CT >= 4 ? 4 : 2;
#pragma unroll
        for (int cg = 0; cg + 1 < CT; cg += G) {
            float v[G][8];
#pragma unroll
            for (int k = 0; k < G; ++k) {
                if (cg + k >= CT) break;
                const float *a = in + (int64_t)(cg + k) * n;
                v[k][0] = __ldg(a + r00);
                v[k][1] = __ldg(a + r00 + 1);
                v[k][2] = __ldg(a + r10);
                v[k][3] = __ldg(a + r10 + 1);
                v[k][4] = __ldg(a + r01);
                v[k][5] = __ldg(a + r01 + 1);
                v[k][6] = __ldg(a + r11);
                v[k][7] = __ldg(a + r11 + 1);
            }
#pragma unroll
        for (int ch = cg; ch + 1 < CT && ch < cg + G; ch += 2) {
            const int k = ch - cg;
            const float2 v000 = make_float2(v[k][0], v[k + 1][0]);
            const float2 v100 = make_float2(v[k][1], v[k + 1][1]);
            const float2 v010 = make_float2(v[k][2], v[k + 1][2]);
            const float2 v110 = make_float2(v[k][3], v[k + 1][3]);
            const float2 v001 = make_float2(v[k][4], v[k + 1][4]);
            const float2 v101 = make_float2(v[k][5], v[k + 1][5]);
            const float2 v011 = make_float2(v[k][6], v[k + 1][6]);
            const float2 v111 = make_float2(v[k][7], v[k + 1][7]);
            const float2 c0 = lerp2(lerp2(v000, v100, GX, FX), lerp2(v010, v110, GX, FX), GY, FY);
            const float2 c1 = lerp2(lerp2(v001, v101, GX, FX), lerp2(v011, v111, GX, FX), GY, FY);
            const float2 r = lerp2(c0, c1, GZ, FZ);
            out[(int64_t)ch * m + vi] = r.x;
            out[(int64_t)(ch + 1) * m + vi] = r.y;
        }
        }
        if (CT & 1) {
            const int ch = CT - 1;
            out[(int64_t)ch * m + vi] = lerp_oct(load_oct(in + (int64_t)ch * n, c), c);
        }
    } else {
        for (int ch = 0; ch < C; ++ch) out[ch * m + vi] = sample(in + ch * n, c);
    }
}

// Warp-level merge of x-adjacent scatter targets: lanes hold x-consecutive
// voxels, so for a smooth field lane t's x1 corner is usually lane t+1's x0
// corner.  `in` = this lane absorbs lane t-1's x1 term, `out` = lane t+1
// absorbed this lane's x1 term (row offsets r are channel independent).
struct XMerge {
    bool in[4], out[4];
};
__device__ __forceinline__ void xmerge_row(int r, bool ok, bool &in, bool &out) {
    const int lane = threadIdx.x & 31;
    const int key = ok ? r : -2 - lane;  // invalid lanes never match
    const int up = __shfl_up_sync(0xffffffffu, ok ? r + 1 : -1, 1);
    in = lane > 0 && ok && up == key;
    out = __shfl_down_sync(0xffffffffu, (int)in, 1) != 0 && lane < 31;
}
// predicated fp32 reduction: no branch around each scatter target
__device__ __forceinline__ void red_if(float *a, float v, bool p) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q red.global.add.f32 [%0], %1;\n}\n" ::"l"(a),
        "f"(v), "r"((int)p)
        : "memory");
}
__device__ __forceinline__ void scatter_row2(float *ia, float *ib, bool two, bool ok, int r,
                                             float2 t0, float2 t1, bool in, bool out) {
    const float nx = __shfl_up_sync(0xffffffffu, t1.x, 1);
    const float ny = __shfl_up_sync(0xffffffffu, t1.y, 1);
    t0.x = in ? t0.x + nx : t0.x;
    t0.y = in ? t0.y + ny : t0.y;
    float *a = ia + r, *b = ib + r;
    red_if(a, t0.x, ok);
    red_if(a + 1, t1.x, ok && !out);
    if (two) {
        red_if(b, t0.y, ok);
        red_if(b + 1, t1.y, ok && !out);
    }
}

// Deterministic gin (mdg_set_deterministic): a 64-bit fixed-point scatter.
// Channel c's terms are rounded to integers at the scale 2^k_c, k_c chosen from
// max |gout_c| so that a sum of up to 8n terms stays below 2^62 (2^-36 of the
// channel maximum or finer at 7 M voxels), and added with integer REDs: an
// integer sum does not depend on the order the adds arrive in, so gin is
// bit-identical from run to run.  fix_convert_k adds acc * 2^-k_c into gin
// (one rounding of the exact sum).  A channel whose gradient holds Inf/NaN
// has no scale and is scattered in fp32 (NaN propagation as the reference).
struct FixAcc {
    long long *acc;      // C planes of n, zeroed
    const unsigned *mx;  // per channel max |gout| as float bits (fix_maxabs_k)
};
__device__ __forceinline__ bool fix_finite(unsigned mbits) { return mbits < 0x7f800000u; }
__device__ __forceinline__ int fix_exp(unsigned mbits, int64_t n) {
    int e;
    frexpf(__uint_as_float(mbits), &e);  // max |g| < 2^e
    const int hb = 64 - __clzll((unsigned long long)(8 * n));
    return 62 - e - hb;
}
// 2^k as two float factors (k spans about [-100, 211])
__device__ __forceinline__ float2 fix_scale(unsigned mbits, int64_t n) {
    const int k = fix_exp(mbits, n);
    return make_float2(exp2f((float)(k / 2)), exp2f((float)(k - k / 2)));
}
// round(t * 2^k): the power-of-two products are exact
__device__ __forceinline__ long long fix_q(float t, float2 s) {
    return __float2ll_rn(mul_(mul_(t, s.x), s.y));
}
__device__ __forceinline__ void red_fix_if(long long *a, long long v, bool p) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q red.global.add.u64 [%0], %1;\n}\n" ::"l"(a),
        "l"(v), "r"((int)p)
        : "memory");
}
__device__ __forceinline__ void scatter_row2_fix(long long *ia, long long *ib, bool two, bool ok,
                                                 int r, float2 t0, float2 t1, bool in, bool out,
                                                 float2 sa, float2 sb) {
    long long q0a = fix_q(t0.x, sa), q1a = fix_q(t1.x, sa);
    long long q0b = fix_q(t0.y, sb), q1b = fix_q(t1.y, sb);
    const long long na = __shfl_up_sync(0xffffffffu, q1a, 1);
    const long long nb = __shfl_up_sync(0xffffffffu, q1b, 1);
    q0a = in ? q0a + na : q0a;
    q0b = in ? q0b + nb : q0b;
    long long *a = ia + r, *b = ib + r;
    red_fix_if(a, q0a, ok);
    red_fix_if(a + 1, q1a, ok && !out);
    if (two) {
        red_fix_if(b, q0b, ok);
        red_fix_if(b + 1, q1b, ok && !out);
    }
}
__device__ __forceinline__ void scatter_fix(long long *__restrict__ gp, const Corners &c, float g,
                                            float2 s) {
    const int x0 = c.ax.i0, dx = c.ax.i1 - c.ax.i0;
    const float wx0 = sub_(1.0f, c.ax.f), wx1 = c.ax.f;
    const float wy0 = sub_(1.0f, c.ay.f), wy1 = c.ay.f;
    const float wz0 = sub_(1.0f, c.az.f), wz1 = c.az.f;
    long long *r00 = gp + (c.o00 + x0), *r10 = gp + (c.o10 + x0);
    long long *r01 = gp + (c.o01 + x0), *r11 = gp + (c.o11 + x0);
    red_fix_if(r00, fix_q(mul_(mul_(mul_(g, wx0), wy0), wz0), s), true);
    red_fix_if(r00 + dx, fix_q(mul_(mul_(mul_(g, wx1), wy0), wz0), s), true);
    red_fix_if(r10, fix_q(mul_(mul_(mul_(g, wx0), wy1), wz0), s), true);
    red_fix_if(r10 + dx, fix_q(mul_(mul_(mul_(g, wx1), wy1), wz0), s), true);
    red_fix_if(r01, fix_q(mul_(mul_(mul_(g, wx0), wy0), wz1), s), true);
    red_fix_if(r01 + dx, fix_q(mul_(mul_(mul_(g, wx1), wy0), wz1), s), true);
    red_fix_if(r11, fix_q(mul_(mul_(mul_(g, wx0), wy1), wz1), s), true);
    red_fix_if(r11 + dx, fix_q(mul_(mul_(mul_(g, wx1), wy1), wz1), s), true);
}

// --------------------------------------------------------------- warp bwd
// sampling.hpp:139-167 (gfield: same per-channel order => bit-exact)
// rbits (nullable): atomicMax of max |phi| over the voxels (float bits), the
// displacement bound the deterministic gin gather needs (warp_gather.cu).
// far_only: this launch is the gather's fallback scatter and runs only when
// that bound exceeds the gather's reach (else every thread returns at once).
template <int CT, bool COMPOSE = false, bool SLAB = false, bool FIX = false>
#ifndef MDG_WBWD_MINB
#define MDG_WBWD_MINB 5
#endif
#ifndef MDG_WBWD_MINB16
#define MDG_WBWD_MINB16 4
#endif
// (the slab form's extra strides and window test, and the fixed-point
// scatter's 64-bit terms, need more registers)
__global__ void __launch_bounds__(kSB, (SLAB || FIX) ? (CT == 16 ? 3 : CT == 8 ? 4 : 5)
                                       : CT == 16 ? MDG_WBWD_MINB16
                                       : (CT == 3 || CT == 8) ? MDG_WBWD_MINB : 5)
warp_bwd_k(const float *__restrict__ in, int C, int h, int w, int l,
           const float *__restrict__ field, const float *__restrict__ gout,
           float *__restrict__ gin, float *__restrict__ gfield, int64_t pb, int64_t pe,
           WarpWin win, unsigned *__restrict__ rbits = nullptr, bool far_only = false,
           FixAcc fxa = FixAcc{nullptr, nullptr}) {
    if (far_only && __uint_as_float(*rbits) <= (float)kGatherReach) return;
    // in/gin and field/gout/gfield channel strides (SLAB: WarpWin)
    const int64_t n = SLAB ? win.csi : (int64_t)h * w * l, m = SLAB ? win.csv : n;
    const int64_t p0 = pb + (int64_t)blockIdx.x * kSB + threadIdx.x;  // voxels [pb, pe)
    // CT > 0 keeps every lane alive for the warp-level scatter merge
    bool ok = p0 < pe;
    if (CT == 0 && !ok && !rbits) return;
    const int64_t p = ok ? p0 : (SLAB ? pb : 0), vi = SLAB ? p - win.vo : p;
    int x, y, z;
    xyz_of(p, h, w, x, y, z);
    const float phx = __ldg(field + vi), phy = __ldg(field + m + vi), phz = __ldg(field + 2 * m + vi);
    if (rbits && !far_only) {
        float m = ok ? fmaxf(fabsf(phx), fmaxf(fabsf(phy), fabsf(phz))) : 0.0f;
        // a NaN entry (fmaxf would drop it) ranks above every bound
        if (ok && (isnan(phx) || isnan(phy) || isnan(phz))) m = __uint_as_float(0x7fc00000u);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            m = __uint_as_float(max(__float_as_uint(m),
                                    __shfl_xor_sync(0xffffffffu, __float_as_uint(m), o)));
        if ((threadIdx.x & 31) == 0) atomicMax(rbits, __float_as_uint(m));
    }
    if (CT == 0 && (!ok || (!gin && !gfield))) return;
    Corners c = corners_at(add_((float)x, phx), add_((float)y, phy), add_((float)z, phz), h, w, l);
    if (SLAB && !in_window(c, win)) {
        if (CT == 0) return;
        ok = false;
        c.o00 = c.o10 = c.o01 = c.o11 = 0;
        c.ax.i0 = 0;
    }
    float gx = 0.0f, gy = 0.0f, gz = 0.0f;
    if (CT > 0) {
        // channel pairs; corner rows as 32-bit element offsets (x1 = x0 + 1;
        // the launcher routes h == 1, where x1 == x0, to the CT == 0 kernel)
        const int r00 = c.o00 + c.ax.i0, r10 = c.o10 + c.ax.i0;
        const int r01 = c.o01 + c.ax.i0, r11 = c.o11 + c.ax.i0;
        XMerge mg;
        if (gin || FIX) {
            xmerge_row(r00, ok, mg.in[0], mg.out[0]);
            xmerge_row(r10, ok, mg.in[1], mg.out[1]);
            xmerge_row(r01, ok, mg.in[2], mg.out[2]);
            xmerge_row(r11, ok, mg.in[3], mg.out[3]);
        }
        const float fx = c.ax.f, fy = c.ay.f, fz = c.az.f;
        const float gxw = sub_(1.0f, fx), gyw = sub_(1.0f, fy), gzw = sub_(1.0f, fz);
        const float2 FX = make_float2(fx, fx), GX = make_float2(gxw, gxw);
        const float2 FY = make_float2(fy, fy), GY = make_float2(gyw, gyw);
        const float2 FZ = make_float2(fz, fz), GZ = make_float2(gzw, gzw);
        const bool lx = c.ax.live, ly = c.ay.live, lz = c.az.live;
        // scalar _rn per lane (see warp_fwd_k: packed ops would be fused)
        auto m2 = [](float2 a, float2 b) { return make_float2(mul_(a.x, b.x), mul_(a.y, b.y)); };
        auto a2 = [](float2 a, float2 b) { return make_float2(add_(a.x, b.x), add_(a.y, b.y)); };
        auto s2 = [](float2 a, float2 b) { return make_float2(sub_(a.x, b.x), sub_(a.y, b.y)); };
        // every channel's upstream gradient up front: loads cannot move across
        // the scatter's atomics, so loading per channel pair would expose one
        // memory latency per pair
        float gv[CT > 0 ? CT : 1];
#pragma unroll
        for (int ch = 0; ch < CT; ++ch) gv[ch] = __ldg(gout + (int64_t)ch * m + vi);
        // phase 1, gfield: loads and arithmetic only (no atomics in between,
        // so corner loads of different channel pairs can be in flight together)
#pragma unroll
        for (int ch = 0; ch < CT; ch += 2) {
            const bool two = ch + 1 < CT;
            const float *a = in + (int64_t)ch * n, *b = two ? a + n : a;
            const float ga = gv[ch];
            const float gb = two ? gv[ch + 1] : 0.0f;
            if (gfield) {
                const float2 v000 = make_float2(__ldg(a + r00), __ldg(b + r00));
                const float2 v100 = make_float2(__ldg(a + r00 + 1), __ldg(b + r00 + 1));
                const float2 v010 = make_float2(__ldg(a + r10), __ldg(b + r10));
                const float2 v110 = make_float2(__ldg(a + r10 + 1), __ldg(b + r10 + 1));
                const float2 v001 = make_float2(__ldg(a + r01), __ldg(b + r01));
                const float2 v101 = make_float2(__ldg(a + r01 + 1), __ldg(b + r01 + 1));
                const float2 v011 = make_float2(__ldg(a + r11), __ldg(b + r11));
                const float2 v111 = make_float2(__ldg(a + r11 + 1), __ldg(b + r11 + 1));
                // sampling.hpp:89-97 per lane
                const float2 zero = make_float2(0.0f, 0.0f);
                const float2 cgx =
                    lx ? a2(m2(a2(m2(s2(v100, v000), GY), m2(s2(v110, v010), FY)), GZ),
                            m2(a2(m2(s2(v101, v001), GY), m2(s2(v111, v011), FY)), FZ))
                       : zero;
                const float2 cgy =
                    ly ? a2(m2(a2(m2(s2(v010, v000), GX), m2(s2(v110, v100), FX)), GZ),
                            m2(a2(m2(s2(v011, v001), GX), m2(s2(v111, v101), FX)), FZ))
                       : zero;
                const float2 cgz =
                    lz ? a2(m2(a2(m2(s2(v001, v000), GX), m2(s2(v101, v100), FX)), GY),
                            m2(a2(m2(s2(v011, v010), GX), m2(s2(v111, v110), FX)), FY))
                       : zero;
                // channel order preserved: a, then b
                if (ga != 0.0f) {
                    gx = add_(gx, mul_(ga, cgx.x));
                    gy = add_(gy, mul_(ga, cgy.x));
                    gz = add_(gz, mul_(ga, cgz.x));
                }
                if (two && gb != 0.0f) {
                    gx = add_(gx, mul_(gb, cgx.y));
                    gy = add_(gy, mul_(gb, cgy.y));
                    gz = add_(gz, mul_(gb, cgz.y));
                }
            }
        }
        // phase 2, gin: the 8-corner scatter
#pragma unroll
        for (int ch = 0; ch < CT; ch += 2) {
            const bool two = ch + 1 < CT;
            const float ga = gv[ch];
            const float gb = two ? gv[ch + 1] : 0.0f;
            const float2 g2 = make_float2(ga, gb);
            // FIX: the pair's fixed-point scales (uniform branch: a non-finite
            // channel sends the pair to the fp32 scatter)
            const unsigned mba = FIX ? __ldg(fxa.mx + ch) : 0u;
            const unsigned mbb = FIX && two ? __ldg(fxa.mx + ch + 1) : 0u;
            // (a lone last channel counts as its own pair partner)
            const bool fa = FIX && fix_finite(mba), fb = two ? FIX && fix_finite(mbb) : fa;
            const bool fixp = fa && fb;
            if (gin || FIX) {
                // terms ((g*wx)*wy)*wz exactly as sampling.hpp:110-117, with the
                // shared prefixes computed once
                const float2 gx0 = m2(g2, GX), gx1 = m2(g2, FX);
                const float2 g00 = m2(gx0, GY), g10 = m2(gx1, GY), g01 = m2(gx0, FY),
                             g11 = m2(gx1, FY);
                const float2 t000 = m2(g00, GZ), t100 = m2(g10, GZ), t010 = m2(g01, GZ),
                             t110 = m2(g11, GZ), t001 = m2(g00, FZ), t101 = m2(g10, FZ),
                             t011 = m2(g01, FZ), t111 = m2(g11, FZ);
                // (a zero gradient gives exact zero terms: the reference's skip
                // of g == 0 channels, sampling.hpp:152, changes nothing)
                if (fixp) {
                    const float2 sa = fix_scale(mba, n), sb = two ? fix_scale(mbb, n) : sa;
                    long long *ia = fxa.acc + (int64_t)ch * n, *ib = ia + n;
                    scatter_row2_fix(ia, ib, two, ok, r00, t000, t100, mg.in[0], mg.out[0], sa, sb);
                    scatter_row2_fix(ia, ib, two, ok, r10, t010, t110, mg.in[1], mg.out[1], sa, sb);
                    scatter_row2_fix(ia, ib, two, ok, r01, t001, t101, mg.in[2], mg.out[2], sa, sb);
                    scatter_row2_fix(ia, ib, two, ok, r11, t011, t111, mg.in[3], mg.out[3], sa, sb);
                } else if (FIX && fa != fb) {
                    // one channel of the pair finite, the other not: each alone
                    auto sw = [](float2 v) { return make_float2(v.y, v.x); };
                    const int rr[4] = {r00, r10, r01, r11};
                    const float2 t0s[4] = {t000, t010, t001, t011}, t1s[4] = {t100, t110, t101, t111};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 u0 = fa ? t0s[q] : sw(t0s[q]), u1 = fa ? t1s[q] : sw(t1s[q]);
                        const float2 v0 = sw(u0), v1 = sw(u1);
                        const int cf = fa ? ch : ch + 1, cn = fa ? ch + 1 : ch;
                        const float2 sf = fix_scale(fa ? mba : mbb, n);
                        scatter_row2_fix(fxa.acc + (int64_t)cf * n, nullptr, false, ok, rr[q], u0, u1,
                                         mg.in[q], mg.out[q], sf, sf);
                        scatter_row2(gin + (int64_t)cn * n, nullptr, false, ok, rr[q], v0, v1,
                                     mg.in[q], mg.out[q]);
                    }
                } else {
                    float *ia = gin + (int64_t)ch * n, *ib = ia + n;
                    scatter_row2(ia, ib, two, ok, r00, t000, t100, mg.in[0], mg.out[0]);
                    scatter_row2(ia, ib, two, ok, r10, t010, t110, mg.in[1], mg.out[1]);
                    scatter_row2(ia, ib, two, ok, r01, t001, t101, mg.in[2], mg.out[2]);
                    scatter_row2(ia, ib, two, ok, r11, t011, t111, mg.in[3], mg.out[3]);
                }
            }
        }
    } else {
        for (int ch = 0; ch < C; ++ch) {
            const float g = __ldg(gout + ch * m + vi);
            if (g == 0.0f) continue;
            const unsigned mb = FIX ? __ldg(fxa.mx + ch) : 0u;
            if (FIX && fix_finite(mb)) scatter_fix(fxa.acc + ch * n, c, g, fix_scale(mb, n));
            else if (gin) scatter(gin + ch * n, c, g);
            if (gfield) {
                float cg[3];
                sample_grad(in + ch * n, c, cg);
                gx = add_(gx, mul_(g, cg[0]));
                gy = add_(gy, mul_(g, cg[1]));
                gz = add_(gz, mul_(g, cg[2]));
            }
        }
    }
    if (gfield && ok) {
        if (COMPOSE) {
            // op_compose = op_add(res, op_warp(prev, res)) (ops.hpp:295-298): the
            // add node replays first (gres += gout), then the warp adds its
            // coordinate gradient (tape.hpp:146-156)
            gfield[vi] = add_(add_(gfield[vi], __ldg(gout + vi)), gx);
            gfield[m + vi] = add_(add_(gfield[m + vi], __ldg(gout + m + vi)), gy);
            gfield[2 * m + vi] = add_(add_(gfield[2 * m + vi], __ldg(gout + 2 * m + vi)), gz);
        } else {
            gfield[vi] = add_(gfield[vi], gx);
            gfield[m + vi] = add_(gfield[m + vi], gy);
            gfield[2 * m + vi] = add_(gfield[2 * m + vi], gz);
        }
    }
}

// channel counts with an unrolled instantiation (the pyramid's C = 1, 3, 8,
// 16, ...); others use the runtime loop
#define MDG_UNPACK(...) __VA_ARGS__
#define MDG_WARP_DISPATCH_T(KERNEL, TA, C, CFG, ARGS)                     \
    switch (C) {                                                           \
        case 1: KERNEL<1, MDG_UNPACK TA><<<MDG_UNPACK CFG>>> ARGS; break;   \
        case 2: KERNEL<2, MDG_UNPACK TA><<<MDG_UNPACK CFG>>> ARGS; break;   \
        case 3: KERNEL<3, MDG_UNPACK TA><<<MDG_UNPACK CFG>>> ARGS; break;   \
        case 4: KERNEL<4, MDG_UNPACK TA><<<MDG_UNPACK CFG>>> ARGS; break;   \
        case 8: KERNEL<8, MDG_UNPACK TA><<<MDG_UNPACK CFG>>> ARGS; break;   \
        case 16: KERNEL<16, MDG_UNPACK TA><<<MDG_UNPACK CFG>>> ARGS; break; \
        default: KERNEL<0, MDG_UNPACK TA><<<MDG_UNPACK CFG>>> ARGS; break;  \
    }
#define MDG_WARP_DISPATCH(KERNEL, C, CFG, ARGS)                  \
    switch (C) {                                                 \
        case 1: KERNEL<1><<<MDG_UNPACK CFG>>> ARGS; break;       \
        case 2: KERNEL<2><<<MDG_UNPACK CFG>>> ARGS; break;       \
        case 3: KERNEL<3><<<MDG_UNPACK CFG>>> ARGS; break;       \
        case 4: KERNEL<4><<<MDG_UNPACK CFG>>> ARGS; break;       \
        case 8: KERNEL<8><<<MDG_UNPACK CFG>>> ARGS; break;       \
        case 16: KERNEL<16><<<MDG_UNPACK CFG>>> ARGS; break;     \
        default: KERNEL<0><<<MDG_UNPACK CFG>>> ARGS; break;      \
    }

// ------------------------------------------------------------ compose fwd
// field_ops.hpp:42-49 / ops.hpp:295-298: out = res + prev(x + res(x))
__global__ void __launch_bounds__(kSB)
compose_fwd_k(const float *__restrict__ prev, const float *__restrict__ res, int h, int w,
              int l, float *__restrict__ out) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (p >= n) return;
    int x, y, z;
    xyz_of(p, h, w, x, y, z);
    const float r0 = __ldg(res + p), r1 = __ldg(res + n + p), r2 = __ldg(res + 2 * n + p);
    const Corners c = corners_at(add_((float)x, r0), add_((float)y, r1), add_((float)z, r2), h, w, l);
    out[p] = add_(sample(prev, c), r0);
    out[n + p] = add_(sample(prev + n, c), r1);
    out[2 * n + p] = add_(sample(prev + 2 * n, c), r2);
}

// ------------------------------------------------------------ compose bwd
// tape order (tape.hpp:146-156 then ops.hpp:285-289): gres += gout, then the
// warp backward adds the coordinate gradient; gprev receives the scatter.
__global__ void __launch_bounds__(kSB)
compose_bwd_k(const float *__restrict__ prev, const float *__restrict__ res, int h, int w,
              int l, const float *__restrict__ gout, float *__restrict__ gprev,
              float *__restrict__ gres) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (p >= n) return;
    int x, y, z;
    xyz_of(p, h, w, x, y, z);
    const float r0 = __ldg(res + p), r1 = __ldg(res + n + p), r2 = __ldg(res + 2 * n + p);
    const Corners c = corners_at(add_((float)x, r0), add_((float)y, r1), add_((float)z, r2), h, w, l);
    float gx = 0.0f, gy = 0.0f, gz = 0.0f;
    float go[3];
    for (int ch = 0; ch < 3; ++ch) {
        const float g = __ldg(gout + ch * n + p);
        go[ch] = g;
        if (g == 0.0f) continue;
        if (gprev) scatter(gprev + ch * n, c, g);
        if (gres) {
            float cg[3];
            sample_grad(prev + ch * n, c, cg);
            gx = add_(gx, mul_(g, cg[0]));
            gy = add_(gy, mul_(g, cg[1]));
            gz = add_(gz, mul_(g, cg[2]));
        }
    }
    if (gres) {
        gres[p] = add_(add_(gres[p], go[0]), gx);
        gres[n + p] = add_(add_(gres[n + p], go[1]), gy);
        gres[2 * n + p] = add_(add_(gres[2 * n + p], go[2]), gz);
    }
}

// ----------------------------------------------------------- upsample fwd
// sampling.hpp:225-242: fine voxel t samples coarse coordinate t/2, * scale
__global__ void __launch_bounds__(kSB)
upsample2_fwd_k(const float *__restrict__ in, int C, int h, int w, int l, int th, int tw,
                int tl, float scale, float *__restrict__ out) {
    const int64_t no = (int64_t)th * tw * tl, ni = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (p >= no) return;
    int x, y, z;
    xyz_of(p, th, tw, x, y, z);
    const Corners c = corners_at((float)x / 2.0f, (float)y / 2.0f, (float)z / 2.0f, h, w, l);
    if (C == 3) {  // the displacement field: the three channels' loads in flight together
        const Oct o0 = load_oct(in, c), o1 = load_oct(in + ni, c), o2 = load_oct(in + 2 * ni, c);
        out[p] = mul_(scale, lerp_oct(o0, c));
        out[no + p] = mul_(scale, lerp_oct(o1, c));
        out[2 * no + p] = mul_(scale, lerp_oct(o2, c));
        return;
    }
    for (int ch = 0; ch < C; ++ch) out[ch * no + p] = mul_(scale, sample(in + ch * ni, c));
}

// The fine positions t = 2i-2 .. 2i+2 on one axis and the corner weight of
// coarse index i in each (the reference scatter's 1-f for i0, f for i1; 0
// when t does not reach i or lies outside the grid).  Fixed-size, fully
// unrolled: no local-memory arrays.
constexpr int kUpTaps = 5;
__device__ __forceinline__ float axis_tap(int i, int k, int dim, int tdim, int &t) {
    t = 2 * i - 2 + k;
    float wgt = 0.0f;
    if (t >= 0 && t < tdim) {
        const Ax a = resolve_axis((float)t / 2.0f, dim);
        // (a collapsed axis has i0 == i1 with f = 0: the reference adds the
        // i1 term g*0 after the i0 term, which changes nothing)
        if (a.i0 == i) wgt = sub_(1.0f, a.f);
        else if (a.i1 == i) wgt = a.f;
    }
    return wgt;
}

// sampling.hpp:245-262 as a gather onto each coarse voxel
__global__ void __launch_bounds__(kSB)
upsample2_bwd_k(int C, int h, int w, int l, int th, int tw, int tl, float scale,
                const float *__restrict__ gout, float *__restrict__ gin) {
    const int64_t no = (int64_t)th * tw * tl, ni = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (p >= ni) return;
    int x, y, z;
    xyz_of(p, h, w, x, y, z);
    int tx[kUpTaps];
    float wx[kUpTaps];
#pragma unroll
    for (int e = 0; e < kUpTaps; ++e) wx[e] = axis_tap(x, e, h, th, tx[e]);
    // the reference's terms ((scale*g*wx)*wy)*wz in fine-voxel order (z, y,
    // x ascending); zero-weight taps are skipped, as a gather adds nothing.
    // Channels inside, so each fine row's taps are computed once.
    float acc[4];
    for (int c0 = 0; c0 < C; c0 += 4) {
        const int cn = min(4, C - c0);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = k < cn ? gin[(c0 + k) * ni + p] : 0.0f;
#pragma unroll 1
        for (int a = 0; a < kUpTaps; ++a) {
            int tz;
            const float wz = axis_tap(z, a, l, tl, tz);
            if (wz == 0.0f) continue;
#pragma unroll 1
            for (int b = 0; b < kUpTaps; ++b) {
                int ty;
                const float wy = axis_tap(y, b, w, tw, ty);
                if (wy == 0.0f) continue;
                const int64_t row = ((int64_t)tz * tw + ty) * th;
#pragma unroll
                for (int e = 0; e < kUpTaps; ++e) {
                    if (wx[e] == 0.0f) continue;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (k >= cn) break;
                        const float g = mul_(scale, __ldg(gout + (c0 + k) * no + row + tx[e]));
                        acc[k] = add_(acc[k], mul_(mul_(mul_(g, wx[e]), wy), wz));
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < cn) gin[(c0 + k) * ni + p] = acc[k];
    }
}

__global__ void scale_k(const float *__restrict__ a, int64_t m, float s, float *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (i < m) out[i] = mul_(a[i], s);
}

__global__ void axpy_k(const float *__restrict__ a, int64_t m, float s, float *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (i < m) out[i] = add_(out[i], mul_(a[i], s));
}

__global__ void add2_k(const float *__restrict__ a, const float *__restrict__ b, int64_t m,
                       float *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (i < m) out[i] = add_(a[i], b[i]);
}

// per channel max |g| as float bits (unsigned order = magnitude order; NaN
// ranks above Inf): the fixed-point scale of the deterministic scatter
__global__ void __launch_bounds__(kSB)
fix_maxabs_k(const float *__restrict__ g, int64_t n, unsigned *__restrict__ mx) {
    const float *gc = g + (int64_t)blockIdx.y * n;
    unsigned m = 0u;
    const int64_t stride = (int64_t)gridDim.x * kSB;
    if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
        const float4 *g4 = reinterpret_cast<const float4 *>(gc);
        for (int64_t i = (int64_t)blockIdx.x * kSB + threadIdx.x; i < n / 4; i += stride) {
            const float4 v = __ldg(g4 + i);
            m = max(max(m, __float_as_uint(fabsf(v.x))), __float_as_uint(fabsf(v.y)));
            m = max(max(m, __float_as_uint(fabsf(v.z))), __float_as_uint(fabsf(v.w)));
        }
    } else {
        for (int64_t i = (int64_t)blockIdx.x * kSB + threadIdx.x; i < n; i += stride)
            m = max(m, __float_as_uint(fabsf(__ldg(gc + i))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(mx + blockIdx.y, m);
}

// gin += acc * 2^-k (acc zero: gin untouched, a -0 stays -0)
__device__ __forceinline__ float fix_add(float gin, long long a, float2 inv) {
    return a == 0 ? gin : add_(gin, mul_(mul_(__ll2float_rn(a), inv.x), inv.y));
}
__global__ void __launch_bounds__(kSB)
fix_convert_k(const long long *__restrict__ acc, int64_t n, const unsigned *__restrict__ mx,
              float *__restrict__ gin) {
    const unsigned mb = __ldg(mx + blockIdx.y);
    if (!fix_finite(mb)) return;  // scattered in fp32
    const int k = fix_exp(mb, n);
    const float2 inv = make_float2(exp2f((float)(-(k / 2))), exp2f((float)(-(k - k / 2))));
    const long long *ac = acc + (int64_t)blockIdx.y * n;
    float *gc = gin + (int64_t)blockIdx.y * n;
    const int64_t stride = (int64_t)gridDim.x * kSB;
    if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(gin) & 15) == 0) {
        for (int64_t i = (int64_t)blockIdx.x * kSB + threadIdx.x; i < n / 4; i += stride) {
            const longlong2 a = __ldg(reinterpret_cast<const longlong2 *>(ac) + 2 * i);
            const longlong2 b = __ldg(reinterpret_cast<const longlong2 *>(ac) + 2 * i + 1);
            float4 v = reinterpret_cast<float4 *>(gc)[i];
            v.x = fix_add(v.x, a.x, inv);
            v.y = fix_add(v.y, a.y, inv);
            v.z = fix_add(v.z, b.x, inv);
            v.w = fix_add(v.w, b.y, inv);
            reinterpret_cast<float4 *>(gc)[i] = v;
        }
    } else {
        for (int64_t i = (int64_t)blockIdx.x * kSB + threadIdx.x; i < n; i += stride)
            gc[i] = fix_add(gc[i], __ldg(ac + i), inv);
    }
}

// The deterministic whole-volume gin: max |gout| per channel, the fixed-point
// scatter (`launch` runs warp_bwd_k<..., FIX = true> with the FixAcc), the
// conversion into gin.  Scratch: 8 bytes per gin element; if the pool cannot
// provide it the caller falls back to the per-target gather.
static mdg_status fix_gin_run(long long *acc, unsigned *mx, size_t bytes, const float *gout, int C,
                              int64_t n, float *gin, cudaStream_t st,
                              const std::function<void(const FixAcc &)> &launch) {
    MDG_CUDA_TRY(cudaMemsetAsync(acc, 0, bytes, st));
    const unsigned gx = (unsigned)std::min<int64_t>((n / 4 + kSB - 1) / kSB + 1, 148 * 8);
    fix_maxabs_k<<<dim3(gx, C), kSB, 0, st>>>(gout, n, mx);
    MDG_LAUNCHED();
    launch(FixAcc{acc, mx});
    MDG_LAUNCHED();
    fix_convert_k<<<dim3(gx, C), kSB, 0, st>>>(acc, n, mx, gin);
    MDG_LAUNCHED();
    return MDG_OK;
}
// false: no memory for the accumulator (the caller gathers per target instead)
static bool fix_gin(const float *gout, int C, int64_t n, float *gin, cudaStream_t st,
                    mdg_status *rc, const std::function<void(const FixAcc &)> &launch) {
    Scratch ws;
    const size_t accb = (size_t)C * n * sizeof(long long), bytes = accb + C * sizeof(unsigned);
    const cudaError_t e = ws.alloc(bytes, st);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();  // clear it: the gather path needs no accumulator
        return false;
    }
    if (e != cudaSuccess) {
        *rc = status_from_cuda(e, "fix_gin");
        return true;
    }
    long long *acc = ws.as<long long>();
    unsigned *mx = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(acc) + accb);
    *rc = fix_gin_run(acc, mx, bytes, gout, C, n, gin, st, launch);
    return true;
}

// voxel-range launchers (the host-call pipeline computes z-chunks of a volume
// whose inputs are fully resident)
mdg_status warp_fwd_range(const float *in, int C, mdg_dims3 d, const float *field, float *out,
                          int64_t pb, int64_t pe, cudaStream_t st) {
    if (pe <= pb) return MDG_OK;
    MDG_WARP_DISPATCH(warp_fwd_k, d.h >= 2 ? C : 0, (grid1d(pe - pb, kSB), kSB, 0, st),
                      (in, C, d.h, d.w, d.l, field, out, pb, pe, whole_win(nvox(d), d.l)));
    MDG_LAUNCHED();
    return MDG_OK;
}

// gin by the float-atomic scatter (fast; the summation order at a shared
// corner varies from run to run) unless deterministic mode is on
// (mdg_set_deterministic / MDG_DETERMINISTIC=1): then, for the whole volume,
// by the 64-bit fixed-point scatter (fix_gin; ~1.5x the cost), and for a voxel
// range by the per-target gather of warp_gather.cu (~3x: a range's targets
// are not bounded, the gather's are); both bit-identical from run to run
static bool warp_atomic_mode() { return !deterministic_mode(); }

mdg_status warp_bwd_range(const float *in, int C, mdg_dims3 d, const float *field,
                          const float *gout, float *gin, float *gfield, int64_t pb, int64_t pe,
                          cudaStream_t st) {
    if (pe <= pb) return MDG_OK;
    const int CD = d.h >= 2 ? C : 0;
    mdg_status frc = MDG_OK;
    if (gin && !warp_atomic_mode() && pb == 0 && pe == nvox(d) &&
        fix_gin(gout, C, nvox(d), gin, st, &frc, [&](const FixAcc &fx) {
            MDG_WARP_DISPATCH_T(warp_bwd_k, (false, false, true), CD,
                                (grid1d(pe - pb, kSB), kSB, 0, st),
                                (in, C, d.h, d.w, d.l, field, gout, gin, gfield, pb, pe,
                                 whole_win(nvox(d), d.l), nullptr, false, fx));
        }))
        return frc;
    // (the gather indexes with 32-bit offsets: up to 16 channel planes)
    if (!gin || warp_atomic_mode() || 16 * nvox(d) >= (int64_t(1) << 32) || d.l >= 4096) {
        MDG_WARP_DISPATCH(warp_bwd_k, CD, (grid1d(pe - pb, kSB), kSB, 0, st),
                          (in, C, d.h, d.w, d.l, field, gout, gin, gfield, pb, pe,
                           whole_win(nvox(d), d.l)));
        MDG_LAUNCHED();
        return MDG_OK;
    }
    // 1. gfield (gather, bit-exact) + the displacement bound; 2. gin gathered
    // per target; 3. the atomic scatter only if the bound is out of reach
    Scratch ws;
    MDG_CUDA_TRY(ws.alloc(gin_gather_scratch_words(d) * sizeof(unsigned), st));
    unsigned *rb = ws.as<unsigned>();
    MDG_CUDA_TRY(cudaMemsetAsync(rb, 0, 2 * sizeof(unsigned), st));
    MDG_WARP_DISPATCH(warp_bwd_k, CD, (grid1d(pe - pb, kSB), kSB, 0, st),
                      (in, C, d.h, d.w, d.l, field, gout, nullptr, gfield, pb, pe,
                       whole_win(nvox(d), d.l), rb, false));
    MDG_LAUNCHED();
    if (mdg_status e = warp_gin_gather(field, gout, C, d, gin, pb, pe, rb, rb + 1, st)) return e;
    MDG_WARP_DISPATCH(warp_bwd_k, CD, (grid1d(pe - pb, kSB), kSB, 0, st),
                      (in, C, d.h, d.w, d.l, field, gout, gin, nullptr, pb, pe,
                       whole_win(nvox(d), d.l), rb, true));
    MDG_LAUNCHED();
    return MDG_OK;
}

}  // namespace mdg

using namespace mdg;

static mdg_status check_field_dims(mdg_dims3 d, const char *op) {
    MDG_REQUIRE(dims_ok(d), std::string(op) + ": invalid dims " + dims_str(d));
    return MDG_OK;
}

extern "C" {

mdg_status mdg_warp_fwd(const float *in, int C, mdg_dims3 d, const float *field, float *out,
                        void *stream) {
    if (mdg_status e = check_field_dims(d, "warp")) return e;
    MDG_REQUIRE(C >= 0, "warp: channels must be >= 0");
    const int64_t n = nvox(d);
    if (n == 0 || C == 0) return MDG_OK;
    MDG_REQUIRE(in && field && out, "warp: null pointer");
    // the unrolled kernels assume x1 = x0 + 1, i.e. h >= 2
    return warp_fwd_range(in, C, d, field, out, 0, n, S_(stream));
}

mdg_status mdg_warp_bwd(const float *in, int C, mdg_dims3 d, const float *field,
                        const float *gout, float *gin, float *gfield, void *stream) {
    if (mdg_status e = check_field_dims(d, "warp")) return e;
    MDG_REQUIRE(C >= 0, "warp: channels must be >= 0");
    const int64_t n = nvox(d);
    if (n == 0 || C == 0 || (!gin && !gfield)) return MDG_OK;
    MDG_REQUIRE(in && field && gout, "warp: null pointer");
    return warp_bwd_range(in, C, d, field, gout, gin, gfield, 0, n, S_(stream));
}

mdg_status mdg_warp_fwd_range(const float *in, int C, mdg_dims3 d, const float *field,
                              float *out, int64_t pb, int64_t pe, void *stream) {
    if (mdg_status e = check_field_dims(d, "warp")) return e;
    MDG_REQUIRE(C >= 0, "warp: channels must be >= 0");
    MDG_REQUIRE(0 <= pb && pb <= pe && pe <= nvox(d), "warp: voxel range out of bounds");
    if (pe == pb || C == 0) return MDG_OK;
    MDG_REQUIRE(in && field && out, "warp: null pointer");
    return warp_fwd_range(in, C, d, field, out, pb, pe, S_(stream));
}

mdg_status mdg_warp_bwd_range(const float *in, int C, mdg_dims3 d, const float *field,
                              const float *gout, float *gin, float *gfield, int64_t pb,
                              int64_t pe, void *stream) {
    if (mdg_status e = check_field_dims(d, "warp")) return e;
    MDG_REQUIRE(C >= 0, "warp: channels must be >= 0");
    MDG_REQUIRE(0 <= pb && pb <= pe && pe <= nvox(d), "warp: voxel range out of bounds");
    if (pe == pb || C == 0 || (!gin && !gfield)) return MDG_OK;
    MDG_REQUIRE(in && field && gout, "warp: null pointer");
    return warp_bwd_range(in, C, d, field, gout, gin, gfield, pb, pe, S_(stream));
}

// Depth-slab forms: planes [z0, z1) of a volume of dims d; in / gin hold the
// planes [zi0, zi1) only, field / out / gout / gfield planes [z0, z1) only.
// A field that samples outside [zi0, zi1) is reported (synchronously) as
// MDG_EINVAL and leaves the out-of-window voxels untouched.
static mdg_status check_slab(mdg_dims3 d, int C, int zi0, int zi1, int z0, int z1) {
    if (mdg_status e = check_field_dims(d, "warp slab")) return e;
    MDG_REQUIRE(C >= 0, "warp slab: channels must be >= 0");
    MDG_REQUIRE(0 <= z0 && z0 <= z1 && z1 <= d.l, "warp slab: plane range out of bounds");
    MDG_REQUIRE(0 <= zi0 && zi0 <= z0 && z1 <= zi1 && zi1 <= d.l,
                "warp slab: input window must cover the slab's planes");
    return MDG_OK;
}

// err_dev non-null: the caller's device word collects violations (no sync,
// graph-capturable); null: a scratch word, read back synchronously
static mdg_status slab_run(mdg_dims3 d, int zi0, int zi1, int z0, int z1, cudaStream_t st,
                           unsigned *err_dev,
                           const std::function<void(const WarpWin &)> &launch) {
    const int64_t hw = (int64_t)d.h * d.w;
    if (err_dev) {
        const WarpWin win{(zi1 - zi0) * hw, (z1 - z0) * hw, z0 * hw, zi0, zi1, (int)(zi0 * hw),
                          err_dev};
        launch(win);
        MDG_LAUNCHED();
        return MDG_OK;
    }
    Scratch ws;
    MDG_CUDA_TRY(ws.alloc(sizeof(unsigned), st));
    unsigned *err = ws.as<unsigned>();
    MDG_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(unsigned), st));
    const WarpWin win{(zi1 - zi0) * hw, (z1 - z0) * hw, z0 * hw, zi0, zi1, (int)(zi0 * hw), err};
    launch(win);
    MDG_LAUNCHED();
    unsigned bad = 0;
    MDG_CUDA_TRY(cudaMemcpyAsync(&bad, err, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    MDG_CUDA_TRY(cudaStreamSynchronize(st));
    MDG_REQUIRE(!bad, "warp slab: the field samples planes outside the input window [" +
                          std::to_string(zi0) + ", " + std::to_string(zi1) + ")");
    return MDG_OK;
}

static mdg_status warp_fwd_slab_impl(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                                     const float *field, float *out, int z0, int z1,
                                     unsigned *err_dev, void *stream) {
    if (mdg_status e = check_slab(d, C, zi0, zi1, z0, z1)) return e;
    const int64_t hw = (int64_t)d.h * d.w;
    if (z1 == z0 || C == 0 || hw == 0) return MDG_OK;
    MDG_REQUIRE(in && field && out, "warp slab: null pointer");
    const int64_t pb = z0 * hw, pe = z1 * hw;
    cudaStream_t st = S_(stream);
    return slab_run(d, zi0, zi1, z0, z1, st, err_dev, [&](const WarpWin &win) {
        MDG_WARP_DISPATCH_T(warp_fwd_k, (true), d.h >= 2 ? C : 0,
                            (grid1d(pe - pb, kSB), kSB, 0, st),
                            (in, C, d.h, d.w, d.l, field, out, pb, pe, win));
    });
}

static mdg_status warp_bwd_slab_impl(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                                     const float *field, const float *gout, float *gin,
                                     float *gfield, int z0, int z1, unsigned *err_dev,
                                     void *stream) {
    if (mdg_status e = check_slab(d, C, zi0, zi1, z0, z1)) return e;
    const int64_t hw = (int64_t)d.h * d.w;
    if (z1 == z0 || C == 0 || hw == 0 || (!gin && !gfield)) return MDG_OK;
    MDG_REQUIRE(in && field && gout, "warp slab: null pointer");
    const int64_t pb = z0 * hw, pe = z1 * hw;
    cudaStream_t st = S_(stream);
    // gin by the float-atomic scatter (the deterministic gather works on
    // whole-volume buffers only)
    return slab_run(d, zi0, zi1, z0, z1, st, err_dev, [&](const WarpWin &win) {
        MDG_WARP_DISPATCH_T(warp_bwd_k, (false, true), d.h >= 2 ? C : 0,
                            (grid1d(pe - pb, kSB), kSB, 0, st),
                            (in, C, d.h, d.w, d.l, field, gout, gin, gfield, pb, pe, win));
    });
}

mdg_status mdg_warp_fwd_slab(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                             const float *field, float *out, int z0, int z1, void *stream) {
    return warp_fwd_slab_impl(in, C, d, zi0, zi1, field, out, z0, z1, nullptr, stream);
}

mdg_status mdg_warp_bwd_slab(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                             const float *field, const float *gout, float *gin, float *gfield,
                             int z0, int z1, void *stream) {
    return warp_bwd_slab_impl(in, C, d, zi0, zi1, field, gout, gin, gfield, z0, z1, nullptr,
                              stream);
}

mdg_status mdg_warp_fwd_slab_async(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                                   const float *field, float *out, int z0, int z1,
                                   unsigned *err, void *stream) {
    MDG_REQUIRE(err, "warp slab: null error word");
    return warp_fwd_slab_impl(in, C, d, zi0, zi1, field, out, z0, z1, err, stream);
}

mdg_status mdg_warp_bwd_slab_async(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                                   const float *field, const float *gout, float *gin,
                                   float *gfield, int z0, int z1, unsigned *err, void *stream) {
    MDG_REQUIRE(err, "warp slab: null error word");
    return warp_bwd_slab_impl(in, C, d, zi0, zi1, field, gout, gin, gfield, z0, z1, err, stream);
}

mdg_status mdg_compose_fwd(const float *prev, const float *res, mdg_dims3 d, float *out,
                           void *stream) {
    if (mdg_status e = check_field_dims(d, "compose")) return e;
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(prev && res && out, "compose: null pointer");
    MDG_REQUIRE(out != prev && out != res, "compose: output must not alias an input");
    compose_fwd_k<<<grid1d(n, kSB), kSB, 0, S_(stream)>>>(prev, res, d.h, d.w, d.l, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_compose_bwd(const float *prev, const float *res, mdg_dims3 d,
                           const float *gout, float *gprev, float *gres, void *stream) {
    if (mdg_status e = check_field_dims(d, "compose")) return e;
    const int64_t n = nvox(d);
    if (n == 0 || (!gprev && !gres)) return MDG_OK;
    MDG_REQUIRE(prev && res && gout, "compose: null pointer");
    MDG_REQUIRE(!(gprev && gprev == gres), "compose: gprev and gres must not alias");
    if (d.h >= 2 && gres) {
        // the warp backward with C = 3 plus the add node: gres by the gather
        // kernel, gprev (the scatter) by the fp32 scatter, or in deterministic
        // mode by the fixed-point scatter
        cudaStream_t st = S_(stream);
        mdg_status frc = MDG_OK;
        if (gprev && !warp_atomic_mode() &&
            fix_gin(gout, 3, n, gprev, st, &frc, [&](const FixAcc &fx) {
                warp_bwd_k<3, true, false, true><<<grid1d(n, kSB), kSB, 0, st>>>(
                    prev, 3, d.h, d.w, d.l, res, gout, gprev, gres, 0, n, whole_win(n, d.l),
                    nullptr, false, fx);
            }))
            return frc;
        if (!gprev || warp_atomic_mode() || 16 * n >= (int64_t(1) << 32) || d.l >= 4096) {
            warp_bwd_k<3, true><<<grid1d(n, kSB), kSB, 0, st>>>(prev, 3, d.h, d.w, d.l, res, gout,
                                                                gprev, gres, 0, n,
                                                                whole_win(n, d.l));
            MDG_LAUNCHED();
            return MDG_OK;
        }
        Scratch ws;
        MDG_CUDA_TRY(ws.alloc(gin_gather_scratch_words(d) * sizeof(unsigned), st));
        unsigned *rb = ws.as<unsigned>();
        MDG_CUDA_TRY(cudaMemsetAsync(rb, 0, 2 * sizeof(unsigned), st));
        warp_bwd_k<3, true><<<grid1d(n, kSB), kSB, 0, st>>>(prev, 3, d.h, d.w, d.l, res, gout,
                                                            nullptr, gres, 0, n,
                                                            whole_win(n, d.l), rb, false);
        MDG_LAUNCHED();
        if (mdg_status e = warp_gin_gather(res, gout, 3, d, gprev, 0, n, rb, rb + 1, st)) return e;
        warp_bwd_k<3, true><<<grid1d(n, kSB), kSB, 0, st>>>(prev, 3, d.h, d.w, d.l, res, gout,
                                                            gprev, nullptr, 0, n,
                                                            whole_win(n, d.l), rb, true);
        MDG_LAUNCHED();
        return MDG_OK;
    }
    compose_bwd_k<<<grid1d(n, kSB), kSB, 0, S_(stream)>>>(prev, res, d.h, d.w, d.l, gout, gprev,
                                                          gres);
    MDG_LAUNCHED();
    return MDG_OK;
}

static mdg_status check_up(mdg_dims3 d, mdg_dims3 td) {
    auto ok = [](int in, int out) { return out >= 2 * in - 1 && out <= 2 * in + 1; };
    MDG_REQUIRE(dims_ok(d) && dims_ok(td), "upsample: invalid dims");
    // sampling.hpp:266-271
    MDG_REQUIRE(ok(d.h, td.h) && ok(d.w, td.w) && ok(d.l, td.l),
                "upsample target dims " + dims_str(td) + " not within doubling range of " +
                    dims_str(d));
    return MDG_OK;
}

mdg_status mdg_upsample2_fwd(const float *in, int C, mdg_dims3 d, mdg_dims3 td, float scale,
                             float *out, void *stream) {
    if (mdg_status e = check_up(d, td)) return e;
    const int64_t no = nvox(td);
    if (no == 0 || C == 0) return MDG_OK;
    MDG_REQUIRE(nvox(d) > 0, "upsample: empty input");
    MDG_REQUIRE(in && out, "upsample: null pointer");
    upsample2_fwd_k<<<grid1d(no, kSB), kSB, 0, S_(stream)>>>(in, C, d.h, d.w, d.l, td.h, td.w,
                                                             td.l, scale, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_upsample2_bwd(int C, mdg_dims3 d, mdg_dims3 td, float scale, const float *gout,
                             float *gin, void *stream) {
    if (mdg_status e = check_up(d, td)) return e;
    const int64_t ni = nvox(d);
    if (ni == 0 || C == 0 || !gin) return MDG_OK;
    MDG_REQUIRE(gout, "upsample: null pointer");
    upsample2_bwd_k<<<grid1d(ni, kSB), kSB, 0, S_(stream)>>>(C, d.h, d.w, d.l, td.h, td.w, td.l,
                                                             scale, gout, gin);
    MDG_LAUNCHED();
    return MDG_OK;
}

// reghead.hpp:52-67
mdg_status mdg_scaling_squaring_fwd(const float *vel, mdg_dims3 d, int steps, float *out,
                                    float *saved, void *stream) {
    MDG_REQUIRE(steps >= 1, "scaling_squaring: steps must be >= 1");
    MDG_REQUIRE(steps <= 30, "scaling_squaring: steps must be <= 30");
    if (mdg_status e = check_field_dims(d, "scaling_squaring")) return e;
    const int64_t n = nvox(d), n3 = 3 * n;
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(vel && out, "scaling_squaring: null pointer");
    cudaStream_t st = S_(stream);
    Scratch tmp;
    float *buf = saved;
    if (!buf) {
        MDG_CUDA_TRY(tmp.alloc(2 * n3 * sizeof(float), st));
        buf = tmp.as<float>();
    }
    auto slot = [&](int i) { return saved ? buf + (int64_t)i * n3 : buf + (int64_t)(i & 1) * n3; };
    const float inv = 1.0f / (float)(1 << steps);
    scale_k<<<grid1d(n3, kSB), kSB, 0, st>>>(vel, n3, inv, slot(0));
    MDG_LAUNCHED();
    for (int i = 0; i < steps; ++i) {
        float *dst = (i == steps - 1 && !saved) ? out : slot(i + 1);
        compose_fwd_k<<<grid1d(n, kSB), kSB, 0, st>>>(slot(i), slot(i), d.h, d.w, d.l, dst);
        MDG_LAUNCHED();
    }
    if (saved)
        MDG_CUDA_TRY(cudaMemcpyAsync(out, slot(steps), n3 * sizeof(float),
                                     cudaMemcpyDeviceToDevice, st));
    return MDG_OK;
}

mdg_status mdg_scaling_squaring_bwd(const float *saved, mdg_dims3 d, int steps,
                                    const float *gout, float *gvel, void *stream) {
    MDG_REQUIRE(steps >= 1 && steps <= 30, "scaling_squaring: steps out of range");
    if (mdg_status e = check_field_dims(d, "scaling_squaring")) return e;
    const int64_t n = nvox(d), n3 = 3 * n;
    if (n == 0 || !gvel) return MDG_OK;
    MDG_REQUIRE(saved && gout, "scaling_squaring: null pointer");
    cudaStream_t st = S_(stream);
    Scratch tmp;
    MDG_CUDA_TRY(tmp.alloc(3 * n3 * sizeof(float), st));
    float *g = tmp.as<float>(), *ga = g + n3, *gb = g + 2 * n3;
    MDG_CUDA_TRY(cudaMemcpyAsync(g, gout, n3 * sizeof(float), cudaMemcpyDeviceToDevice, st));
    for (int i = steps - 1; i >= 0; --i) {
        // phi_{i+1} = compose(phi_i, phi_i): both operands receive gradient
        MDG_CUDA_TRY(cudaMemsetAsync(ga, 0, 2 * n3 * sizeof(float), st));
        const float *phi = saved + (int64_t)i * n3;
        compose_bwd_k<<<grid1d(n, kSB), kSB, 0, st>>>(phi, phi, d.h, d.w, d.l, g, ga, gb);
        MDG_LAUNCHED();
        add2_k<<<grid1d(n3, kSB), kSB, 0, st>>>(ga, gb, n3, g);
        MDG_LAUNCHED();
    }
    axpy_k<<<grid1d(n3, kSB), kSB, 0, st>>>(g, n3, 1.0f / (float)(1 << steps), gvel);
    MDG_LAUNCHED();
    return MDG_OK;
}

}  // extern "C"
