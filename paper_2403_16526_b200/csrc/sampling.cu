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
#include "mdg_common.cuh"

namespace mdg {

constexpr int kSB = 256;

struct Corners {
    Ax ax, ay, az;
    int64_t o00, o10, o01, o11;  // plane offsets of the (y,z) corner rows
};

__device__ __forceinline__ Corners corners_at(float cx, float cy, float cz, int h, int w, int l) {
    Corners c;
    c.ax = resolve_axis(cx, h);
    c.ay = resolve_axis(cy, w);
    c.az = resolve_axis(cz, l);
    const int64_t sy = h, sz = (int64_t)h * w;
    c.o00 = c.az.i0 * sz + c.ay.i0 * sy;
    c.o10 = c.az.i0 * sz + c.ay.i1 * sy;
    c.o01 = c.az.i1 * sz + c.ay.i0 * sy;
    c.o11 = c.az.i1 * sz + c.ay.i1 * sy;
    return c;
}

// sampling.hpp:53-68
__device__ __forceinline__ float sample(const float *__restrict__ pl, const Corners &c) {
    const int x0 = c.ax.i0, x1 = c.ax.i1;
    const float fx = c.ax.f;
    const float c00 = lerp_(__ldg(pl + c.o00 + x0), __ldg(pl + c.o00 + x1), fx);
    const float c10 = lerp_(__ldg(pl + c.o10 + x0), __ldg(pl + c.o10 + x1), fx);
    const float c01 = lerp_(__ldg(pl + c.o01 + x0), __ldg(pl + c.o01 + x1), fx);
    const float c11 = lerp_(__ldg(pl + c.o11 + x0), __ldg(pl + c.o11 + x1), fx);
    const float c0 = lerp_(c00, c10, c.ay.f);
    const float c1 = lerp_(c01, c11, c.ay.f);
    return lerp_(c0, c1, c.az.f);
}

// sampling.hpp:73-99 (zero on dead axes)
__device__ __forceinline__ void sample_grad(const float *__restrict__ pl, const Corners &c,
                                            float g[3]) {
    const int x0 = c.ax.i0, x1 = c.ax.i1;
    const float v000 = __ldg(pl + c.o00 + x0), v100 = __ldg(pl + c.o00 + x1);
    const float v010 = __ldg(pl + c.o10 + x0), v110 = __ldg(pl + c.o10 + x1);
    const float v001 = __ldg(pl + c.o01 + x0), v101 = __ldg(pl + c.o01 + x1);
    const float v011 = __ldg(pl + c.o11 + x0), v111 = __ldg(pl + c.o11 + x1);
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
    const int x0 = c.ax.i0, x1 = c.ax.i1;
    const float wx0 = sub_(1.0f, c.ax.f), wx1 = c.ax.f;
    const float wy0 = sub_(1.0f, c.ay.f), wy1 = c.ay.f;
    const float wz0 = sub_(1.0f, c.az.f), wz1 = c.az.f;
    atomicAdd(gp + c.o00 + x0, mul_(mul_(mul_(g, wx0), wy0), wz0));
    atomicAdd(gp + c.o00 + x1, mul_(mul_(mul_(g, wx1), wy0), wz0));
    atomicAdd(gp + c.o10 + x0, mul_(mul_(mul_(g, wx0), wy1), wz0));
    atomicAdd(gp + c.o10 + x1, mul_(mul_(mul_(g, wx1), wy1), wz0));
    atomicAdd(gp + c.o01 + x0, mul_(mul_(mul_(g, wx0), wy0), wz1));
    atomicAdd(gp + c.o01 + x1, mul_(mul_(mul_(g, wx1), wy0), wz1));
    atomicAdd(gp + c.o11 + x0, mul_(mul_(mul_(g, wx0), wy1), wz1));
    atomicAdd(gp + c.o11 + x1, mul_(mul_(mul_(g, wx1), wy1), wz1));
}

__device__ __forceinline__ void xyz_of(int64_t p, int h, int w, int &x, int &y, int &z) {
    x = (int)(p % h);
    const int64_t t = p / h;
    y = (int)(t % w);
    z = (int)(t / w);
}

// --------------------------------------------------------------- warp fwd
// sampling.hpp:123-135
__global__ void __launch_bounds__(kSB)
warp_fwd_k(const float *__restrict__ in, int C, int h, int w, int l,
           const float *__restrict__ field, float *__restrict__ out) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (p >= n) return;
    int x, y, z;
    xyz_of(p, h, w, x, y, z);
    const Corners c = corners_at(add_((float)x, __ldg(field + p)), add_((float)y, __ldg(field + n + p)),
                                 add_((float)z, __ldg(field + 2 * n + p)), h, w, l);
    for (int ch = 0; ch < C; ++ch) out[ch * n + p] = sample(in + ch * n, c);
}

// --------------------------------------------------------------- warp bwd
// sampling.hpp:139-167
__global__ void __launch_bounds__(kSB)
warp_bwd_k(const float *__restrict__ in, int C, int h, int w, int l,
           const float *__restrict__ field, const float *__restrict__ gout,
           float *__restrict__ gin, float *__restrict__ gfield) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kSB + threadIdx.x;
    if (p >= n) return;
    int x, y, z;
    xyz_of(p, h, w, x, y, z);
    const Corners c = corners_at(add_((float)x, __ldg(field + p)), add_((float)y, __ldg(field + n + p)),
                                 add_((float)z, __ldg(field + 2 * n + p)), h, w, l);
    float gx = 0.0f, gy = 0.0f, gz = 0.0f;
    for (int ch = 0; ch < C; ++ch) {
        const float g = __ldg(gout + ch * n + p);
        if (g == 0.0f) continue;
        if (gin) scatter(gin + ch * n, c, g);
        if (gfield) {
            float cg[3];
            sample_grad(in + ch * n, c, cg);
            gx = add_(gx, mul_(g, cg[0]));
            gy = add_(gy, mul_(g, cg[1]));
            gz = add_(gz, mul_(g, cg[2]));
        }
    }
    if (gfield) {
        gfield[p] = add_(gfield[p], gx);
        gfield[n + p] = add_(gfield[n + p], gy);
        gfield[2 * n + p] = add_(gfield[2 * n + p], gz);
    }
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
    for (int ch = 0; ch < C; ++ch) out[ch * no + p] = mul_(scale, sample(in + ch * ni, c));
}

// fine positions t on one axis whose resolved corners include coarse index i,
// with the corner weight the reference scatter uses (1-f for i0, f for i1)
__device__ __forceinline__ int axis_sources(int i, int dim, int tdim, int *ts, float *ws) {
    int m = 0;
    const int t0 = max(0, 2 * i - 2), t1 = min(tdim - 1, 2 * i + 2);
    for (int t = t0; t <= t1; ++t) {
        const Ax a = resolve_axis((float)t / 2.0f, dim);
        if (a.i0 == i) {
            ts[m] = t;
            ws[m] = sub_(1.0f, a.f);
            ++m;
        }
        if (a.i1 == i) {
            ts[m] = t;
            ws[m] = a.f;
            ++m;
        }
    }
    return m;
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
    int tx[10], ty[10], tz[10];
    float wx[10], wy[10], wz[10];
    const int mx = axis_sources(x, h, th, tx, wx);
    const int my = axis_sources(y, w, tw, ty, wy);
    const int mz = axis_sources(z, l, tl, tz, wz);
    for (int ch = 0; ch < C; ++ch) {
        const float *go = gout + ch * no;
        float acc = gin[ch * ni + p];
        for (int a = 0; a < mz; ++a)
            for (int b = 0; b < my; ++b) {
                const int64_t row = ((int64_t)tz[a] * tw + ty[b]) * th;
                for (int e = 0; e < mx; ++e) {
                    const float g = mul_(scale, __ldg(go + row + tx[e]));
                    acc = add_(acc, mul_(mul_(mul_(g, wx[e]), wy[b]), wz[a]));
                }
            }
        gin[ch * ni + p] = acc;
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
    warp_fwd_k<<<grid1d(n, kSB), kSB, 0, S_(stream)>>>(in, C, d.h, d.w, d.l, field, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_warp_bwd(const float *in, int C, mdg_dims3 d, const float *field,
                        const float *gout, float *gin, float *gfield, void *stream) {
    if (mdg_status e = check_field_dims(d, "warp")) return e;
    MDG_REQUIRE(C >= 0, "warp: channels must be >= 0");
    const int64_t n = nvox(d);
    if (n == 0 || C == 0 || (!gin && !gfield)) return MDG_OK;
    MDG_REQUIRE(in && field && gout, "warp: null pointer");
    warp_bwd_k<<<grid1d(n, kSB), kSB, 0, S_(stream)>>>(in, C, d.h, d.w, d.l, field, gout, gin,
                                                       gfield);
    MDG_LAUNCHED();
    return MDG_OK;
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
