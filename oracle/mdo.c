/*
 * mdo.c — CPU ORACLE (test infrastructure only; see mdo.h).
 *
 * Plain-C restatement of the reference's hot-path loops.  Each function cites
 * the reference file:line (relative to /root/reference/proj/include/mdreg/) it
 * restates.  Arithmetic is written in the reference's evaluation order and the
 * file is compiled with -ffp-contract=off, so with the same libm the results
 * are bit-identical to the reference compiled the same way (checked by
 * tests/test_oracle.py against oracle/_ref and the golden fixtures).
 */
#include "mdo.h"

#include <math.h>
#include <stddef.h>
#include <stdlib.h>

/* ---------------------------------------------------------------- indexing */

/* common.hpp:56-59: x fastest, then y, then z */
static inline int64_t vidx(int h, int w, int x, int y, int z) {
    return ((int64_t)z * w + y) * h + x;
}

/* common.hpp:61-63 */
static inline int inb(int h, int w, int l, int x, int y, int z) {
    return x >= 0 && x < h && y >= 0 && y < w && z >= 0 && z < l;
}

/* --------------------------------------------------------------------- rng */

void mdo_rng_init(mdo_rng *r, uint64_t seed) {
    r->state = seed;
    r->has_spare = 0;
    r->spare = 0.0;
}

/* rng.hpp:27-32 splitmix64 step */
uint64_t mdo_rng_next_u64(mdo_rng *r) {
    r->state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = r->state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:35-37: top 53 bits scaled to [0,1) */
double mdo_rng_uniform01(mdo_rng *r) {
    return (double)(mdo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:39 */
double mdo_rng_uniform(mdo_rng *r, double lo, double hi) {
    return lo + (hi - lo) * mdo_rng_uniform01(r);
}

/* rng.hpp:41-43 (inclusive bounds) */
int mdo_rng_uniform_int(mdo_rng *r, int lo, int hi) {
    return lo + (int)(mdo_rng_next_u64(r) % (uint64_t)(hi - lo + 1));
}

/* rng.hpp:46-59: Box-Muller, cos branch returned, sin branch cached */
double mdo_rng_normal(mdo_rng *r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = mdo_rng_uniform01(r);
    double u2 = mdo_rng_uniform01(r);
    if (u1 < 1e-300) u1 = 1e-300;
    double rad = sqrt(-2.0 * log(u1));
    double ang = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(ang);
    r->has_spare = 1;
    return rad * cos(ang);
}

void mdo_rng_fill_uniform(mdo_rng *r, float *out, int64_t n, double lo, double hi) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)mdo_rng_uniform(r, lo, hi);
}

/* rng.hpp:61: mean + stddev * normal() */
void mdo_rng_fill_normal(mdo_rng *r, float *out, int64_t n, double mean, double sd) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(mean + sd * mdo_rng_normal(r));
}

/* --------------------------------------------------------------- attention */

/* attention.hpp:57-60: slot o -> (dx,dy,dz), x fastest, components in [-r,r] */
void mdo_window_offset(int o, int nb, int off[3]) {
    int r = (nb - 1) / 2;
    off[0] = o % nb - r;
    off[1] = (o / nb) % nb - r;
    off[2] = o / (nb * nb) - r;
}

/* attention.hpp:65-75: max-subtracted softmax, multiply by 1/sum */
static void softmax_row(float *v, int m) {
    float mx = v[0];
    for (int i = 1; i < m; ++i) mx = (mx < v[i]) ? v[i] : mx;
    float sum = 0.0f;
    for (int i = 0; i < m; ++i) {
        v[i] = expf(v[i] - mx);
        sum += v[i];
    }
    float inv = 1.0f / sum;
    for (int i = 0; i < m; ++i) v[i] *= inv;
}

/* attention.hpp:83-123.  logit(o) = B[s,o] + [in bounds] * <q_p, k_{p+off(o)}>;
 * W[s,p,:] = softmax(logits).  No 1/sqrt(d) scale. */
int mdo_na_fwd(const float *Q, const float *K, const float *B, int h, int w, int l, int S,
               int hd, int nb, float *W, int bad[4]) {
    const int64_t n = (int64_t)h * w * l;
    const int win = nb * nb * nb;
    const int r = (nb - 1) / 2;
    const int SD = S * hd;
    float logits[343]; /* nb <= 7 */
    if (win > 343) return 2;
    for (int s = 0; s < S; ++s) {
        const float *bias = B + (int64_t)s * win;
        int64_t p = 0;
        for (int z = 0; z < l; ++z)
            for (int y = 0; y < w; ++y)
                for (int x = 0; x < h; ++x, ++p) {
                    const float *q = Q + p * SD + (int64_t)s * hd;
                    int o = 0;
                    for (int dz = -r; dz <= r; ++dz)
                        for (int dy = -r; dy <= r; ++dy)
                            for (int dx = -r; dx <= r; ++dx, ++o) {
                                float lg = bias[o];
                                if (inb(h, w, l, x + dx, y + dy, z + dz)) {
                                    const float *k =
                                        K + vidx(h, w, x + dx, y + dy, z + dz) * SD +
                                        (int64_t)s * hd;
                                    float dot = 0.0f;
                                    for (int j = 0; j < hd; ++j) dot += q[j] * k[j];
                                    lg += dot;
                                }
                                if (!isfinite((double)lg)) {
                                    if (bad) {
                                        bad[0] = x;
                                        bad[1] = y;
                                        bad[2] = z;
                                        bad[3] = s;
                                    }
                                    return 1;
                                }
                                logits[o] = lg;
                            }
                    softmax_row(logits, win);
                    float *dst = W + ((int64_t)s * n + p) * win;
                    for (int i = 0; i < win; ++i) dst[i] = logits[i];
                }
    }
    return 0;
}

/* attention.hpp:127-166.  dl = W*(gW - <W,gW>); gB += dl; for in-bounds
 * neighbours with dl != 0: gQ_p += dl*K_q, gK_q += dl*Q_p. */
void mdo_na_bwd(const float *Q, const float *K, const float *W, int h, int w, int l, int S,
                int hd, int nb, const float *gW, float *gQ, float *gK, float *gB) {
    const int64_t n = (int64_t)h * w * l;
    const int win = nb * nb * nb;
    const int r = (nb - 1) / 2;
    const int SD = S * hd;
    float dl[343];
    for (int s = 0; s < S; ++s) {
        float *gbias = gB + (int64_t)s * win;
        int64_t p = 0;
        for (int z = 0; z < l; ++z)
            for (int y = 0; y < w; ++y)
                for (int x = 0; x < h; ++x, ++p) {
                    const float *wr = W + ((int64_t)s * n + p) * win;
                    const float *gr = gW + ((int64_t)s * n + p) * win;
                    float dot = 0.0f;
                    for (int i = 0; i < win; ++i) dot += wr[i] * gr[i];
                    for (int i = 0; i < win; ++i) dl[i] = wr[i] * (gr[i] - dot);
                    const float *q = Q + p * SD + (int64_t)s * hd;
                    float *gq = gQ + p * SD + (int64_t)s * hd;
                    int o = 0;
                    for (int dz = -r; dz <= r; ++dz)
                        for (int dy = -r; dy <= r; ++dy)
                            for (int dx = -r; dx <= r; ++dx, ++o) {
                                const float d = dl[o];
                                gbias[o] += d;
                                if (d == 0.0f) continue;
                                if (!inb(h, w, l, x + dx, y + dy, z + dz)) continue;
                                const int64_t qi = vidx(h, w, x + dx, y + dy, z + dz);
                                const float *k = K + qi * SD + (int64_t)s * hd;
                                float *gk = gK + qi * SD + (int64_t)s * hd;
                                for (int j = 0; j < hd; ++j) {
                                    gq[j] += d * k[j];
                                    gk[j] += d * q[j];
                                }
                            }
                }
    }
}

/* attention.hpp:282-298: phi[3s+c, p] = sum_o W[s,p,o] * off_c(o) */
void mdo_subfields_fwd(const float *W, int h, int w, int l, int S, int nb, float *out) {
    const int64_t n = (int64_t)h * w * l;
    const int win = nb * nb * nb;
    for (int s = 0; s < S; ++s)
        for (int64_t p = 0; p < n; ++p) {
            const float *wr = W + ((int64_t)s * n + p) * win;
            float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f;
            for (int o = 0; o < win; ++o) {
                int off[3];
                mdo_window_offset(o, nb, off);
                a0 += wr[o] * (float)off[0];
                a1 += wr[o] * (float)off[1];
                a2 += wr[o] * (float)off[2];
            }
            out[((int64_t)s * 3 + 0) * n + p] = a0;
            out[((int64_t)s * 3 + 1) * n + p] = a1;
            out[((int64_t)s * 3 + 2) * n + p] = a2;
        }
}

/* attention.hpp:301-316: gW[s,p,o] += gphi . off(o) */
void mdo_subfields_bwd(int h, int w, int l, int S, int nb, const float *gout, float *gW) {
    const int64_t n = (int64_t)h * w * l;
    const int win = nb * nb * nb;
    for (int s = 0; s < S; ++s)
        for (int64_t p = 0; p < n; ++p) {
            const float gx = gout[((int64_t)s * 3 + 0) * n + p];
            const float gy = gout[((int64_t)s * 3 + 1) * n + p];
            const float gz = gout[((int64_t)s * 3 + 2) * n + p];
            float *gr = gW + ((int64_t)s * n + p) * win;
            for (int o = 0; o < win; ++o) {
                int off[3];
                mdo_window_offset(o, nb, off);
                gr[o] += gx * (float)off[0] + gy * (float)off[1] + gz * (float)off[2];
            }
        }
}

/* attention.hpp:421-427 */
int mdo_rows_normalized(const float *W, int64_t rows, int win, double tol) {
    for (int64_t r = 0; r < rows; ++r) {
        float s = 0.0f;
        for (int o = 0; o < win; ++o) s += W[r * win + o];
        if (fabs((double)s - 1.0) > tol) return 0;
    }
    return 1;
}

/* ---------------------------------------------------------------- sampling */

/* sampling.hpp:38-49: clamp to [0, dim-1]; i0 = floor, capped at dim-2;
 * live only strictly inside (0, dim-1); dim <= 1 collapses the axis. */
void mdo_resolve_axis(float x, int dim, int *i0, int *i1, float *f, int *live) {
    if (dim <= 1) {
        *i0 = 0;
        *i1 = 0;
        *f = 0.0f;
        *live = 0;
        return;
    }
    const float hi = (float)(dim - 1);
    const float xc = x < 0.0f ? 0.0f : (x > hi ? hi : x);
    int a = (int)floorf(xc);
    if (a > dim - 2) a = dim - 2;
    *i0 = a;
    *i1 = a + 1;
    *f = xc - (float)a;
    *live = x > 0.0f && x < hi;
}

typedef struct {
    int i0, i1, live;
    float f;
} axs;

static inline axs resolve(float x, int dim) {
    axs a;
    mdo_resolve_axis(x, dim, &a.i0, &a.i1, &a.f, &a.live);
    return a;
}

/* sampling.hpp:53-68: lerp along x, then y, then z */
static float sample(const float *pl, int h, int w, axs ax, axs ay, axs az) {
    const int64_t sy = h, sz = (int64_t)h * w;
    const float *p00 = pl + az.i0 * sz + ay.i0 * sy;
    const float *p10 = pl + az.i0 * sz + ay.i1 * sy;
    const float *p01 = pl + az.i1 * sz + ay.i0 * sy;
    const float *p11 = pl + az.i1 * sz + ay.i1 * sy;
    const float gx = 1.0f - ax.f, gy = 1.0f - ay.f, gz = 1.0f - az.f;
    const float c00 = p00[ax.i0] * gx + p00[ax.i1] * ax.f;
    const float c10 = p10[ax.i0] * gx + p10[ax.i1] * ax.f;
    const float c01 = p01[ax.i0] * gx + p01[ax.i1] * ax.f;
    const float c11 = p11[ax.i0] * gx + p11[ax.i1] * ax.f;
    const float c0 = c00 * gy + c10 * ay.f;
    const float c1 = c01 * gy + c11 * ay.f;
    return c0 * gz + c1 * az.f;
}

/* sampling.hpp:73-99: d(sample)/d(coords); zero on dead axes */
static void sample_grad(const float *pl, int h, int w, axs ax, axs ay, axs az, float g[3]) {
    const int64_t sy = h, sz = (int64_t)h * w;
    const float v000 = pl[az.i0 * sz + ay.i0 * sy + ax.i0];
    const float v100 = pl[az.i0 * sz + ay.i0 * sy + ax.i1];
    const float v010 = pl[az.i0 * sz + ay.i1 * sy + ax.i0];
    const float v110 = pl[az.i0 * sz + ay.i1 * sy + ax.i1];
    const float v001 = pl[az.i1 * sz + ay.i0 * sy + ax.i0];
    const float v101 = pl[az.i1 * sz + ay.i0 * sy + ax.i1];
    const float v011 = pl[az.i1 * sz + ay.i1 * sy + ax.i0];
    const float v111 = pl[az.i1 * sz + ay.i1 * sy + ax.i1];
    const float fx = ax.f, fy = ay.f, fz = az.f;
    g[0] = g[1] = g[2] = 0.0f;
    if (ax.live)
        g[0] = ((v100 - v000) * (1.0f - fy) + (v110 - v010) * fy) * (1.0f - fz) +
               ((v101 - v001) * (1.0f - fy) + (v111 - v011) * fy) * fz;
    if (ay.live)
        g[1] = ((v010 - v000) * (1.0f - fx) + (v110 - v100) * fx) * (1.0f - fz) +
               ((v011 - v001) * (1.0f - fx) + (v111 - v101) * fx) * fz;
    if (az.live)
        g[2] = ((v001 - v000) * (1.0f - fx) + (v101 - v100) * fx) * (1.0f - fy) +
               ((v011 - v010) * (1.0f - fx) + (v111 - v110) * fx) * fy;
}

/* sampling.hpp:103-118: weighted 8-corner scatter */
static void scatter(float *gp, int h, int w, axs ax, axs ay, axs az, float g) {
    const int64_t sy = h, sz = (int64_t)h * w;
    const float wx0 = 1.0f - ax.f, wx1 = ax.f;
    const float wy0 = 1.0f - ay.f, wy1 = ay.f;
    const float wz0 = 1.0f - az.f, wz1 = az.f;
    gp[az.i0 * sz + ay.i0 * sy + ax.i0] += g * wx0 * wy0 * wz0;
    gp[az.i0 * sz + ay.i0 * sy + ax.i1] += g * wx1 * wy0 * wz0;
    gp[az.i0 * sz + ay.i1 * sy + ax.i0] += g * wx0 * wy1 * wz0;
    gp[az.i0 * sz + ay.i1 * sy + ax.i1] += g * wx1 * wy1 * wz0;
    gp[az.i1 * sz + ay.i0 * sy + ax.i0] += g * wx0 * wy0 * wz1;
    gp[az.i1 * sz + ay.i0 * sy + ax.i1] += g * wx1 * wy0 * wz1;
    gp[az.i1 * sz + ay.i1 * sy + ax.i0] += g * wx0 * wy1 * wz1;
    gp[az.i1 * sz + ay.i1 * sy + ax.i1] += g * wx1 * wy1 * wz1;
}

/* sampling.hpp:123-135: out_c(x) = in_c(x + field(x)); the coordinate is the
 * fp32 sum float(x) + field. */
void mdo_warp_fwd(const float *in, int C, int h, int w, int l, const float *field, float *out) {
    const int64_t n = (int64_t)h * w * l;
    int64_t p = 0;
    for (int z = 0; z < l; ++z)
        for (int y = 0; y < w; ++y)
            for (int x = 0; x < h; ++x, ++p) {
                const axs ax = resolve((float)x + field[p], h);
                const axs ay = resolve((float)y + field[n + p], w);
                const axs az = resolve((float)z + field[2 * n + p], l);
                for (int c = 0; c < C; ++c) out[c * n + p] = sample(in + c * n, h, w, ax, ay, az);
            }
}

/* sampling.hpp:139-167 */
void mdo_warp_bwd(const float *in, int C, int h, int w, int l, const float *field,
                  const float *gout, float *gin, float *gfield) {
    const int64_t n = (int64_t)h * w * l;
    int64_t p = 0;
    for (int z = 0; z < l; ++z)
        for (int y = 0; y < w; ++y)
            for (int x = 0; x < h; ++x, ++p) {
                const axs ax = resolve((float)x + field[p], h);
                const axs ay = resolve((float)y + field[n + p], w);
                const axs az = resolve((float)z + field[2 * n + p], l);
                float gx = 0.0f, gy = 0.0f, gz = 0.0f;
                for (int c = 0; c < C; ++c) {
                    const float g = gout[c * n + p];
                    if (g == 0.0f) continue;
                    if (gin) scatter(gin + c * n, h, w, ax, ay, az, g);
                    if (gfield) {
                        float cg[3];
                        sample_grad(in + c * n, h, w, ax, ay, az, cg);
                        gx += g * cg[0];
                        gy += g * cg[1];
                        gz += g * cg[2];
                    }
                }
                if (gfield) {
                    gfield[p] += gx;
                    gfield[n + p] += gy;
                    gfield[2 * n + p] += gz;
                }
            }
}

/* sampling.hpp:266-271 */
int mdo_upsample_target_ok(int h, int w, int l, int th, int tw, int tl) {
#define MDO_OK2(a, b) ((b) >= 2 * (a) - 1 && (b) <= 2 * (a) + 1)
    return MDO_OK2(h, th) && MDO_OK2(w, tw) && MDO_OK2(l, tl);
#undef MDO_OK2
}

/* sampling.hpp:225-242: output voxel y samples input coordinate y/2, times scale */
void mdo_upsample2_fwd(const float *in, int C, int h, int w, int l, int th, int tw, int tl,
                       float scale, float *out) {
    const int64_t ni = (int64_t)h * w * l, no = (int64_t)th * tw * tl;
    for (int c = 0; c < C; ++c) {
        int64_t o = 0;
        for (int z = 0; z < tl; ++z) {
            const axs az = resolve((float)z / 2.0f, l);
            for (int y = 0; y < tw; ++y) {
                const axs ay = resolve((float)y / 2.0f, w);
                for (int x = 0; x < th; ++x, ++o) {
                    const axs ax = resolve((float)x / 2.0f, h);
                    out[c * no + o] = scale * sample(in + c * ni, h, w, ax, ay, az);
                }
            }
        }
    }
}

/* sampling.hpp:245-262 */
void mdo_upsample2_bwd(int C, int h, int w, int l, int th, int tw, int tl, float scale,
                       const float *gout, float *gin) {
    const int64_t ni = (int64_t)h * w * l, no = (int64_t)th * tw * tl;
    for (int c = 0; c < C; ++c) {
        int64_t o = 0;
        for (int z = 0; z < tl; ++z) {
            const axs az = resolve((float)z / 2.0f, l);
            for (int y = 0; y < tw; ++y) {
                const axs ay = resolve((float)y / 2.0f, w);
                for (int x = 0; x < th; ++x, ++o) {
                    const axs ax = resolve((float)x / 2.0f, h);
                    scatter(gin + c * ni, h, w, ax, ay, az, scale * gout[c * no + o]);
                }
            }
        }
    }
}

/* ------------------------------------------------------------------- conv3 */

/* ops.hpp:58-74 with slab_axpy 27-37: per output element the terms arrive in
 * (ci, dz, dy, dx) order starting from the bias; zero taps are skipped. */
void mdo_conv3_fwd(const float *in, int ic, int h, int w, int l, const float *k,
                   const float *bias, int oc, float *out) {
    const int64_t n = (int64_t)h * w * l;
    for (int co = 0; co < oc; ++co) {
        float *dst = out + (int64_t)co * n;
        for (int64_t i = 0; i < n; ++i) dst[i] = bias ? bias[co] : 0.0f;
        for (int ci = 0; ci < ic; ++ci) {
            const float *src = in + (int64_t)ci * n;
            const float *kk = k + ((int64_t)co * ic + ci) * 27;
            for (int t = 0; t < 27; ++t) {
                const float kv = kk[t];
                if (kv == 0.0f) continue;
                const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
                for (int z = 0; z < l; ++z) {
                    if (z + dz < 0 || z + dz >= l) continue;
                    for (int y = 0; y < w; ++y) {
                        if (y + dy < 0 || y + dy >= w) continue;
                        for (int x = 0; x < h; ++x) {
                            if (x + dx < 0 || x + dx >= h) continue;
                            dst[vidx(h, w, x, y, z)] += kv * src[vidx(h, w, x + dx, y + dy, z + dz)];
                        }
                    }
                }
            }
        }
    }
}

/* ops.hpp:77-99 with slab_dot 40-53: gbias += sum(gout); gk += correlation of
 * gout with the shifted input; gin += kv * gout shifted back (nonzero taps). */
void mdo_conv3_bwd(const float *in, int ic, int h, int w, int l, const float *k, int oc,
                   const float *gout, float *gin, float *gk, float *gbias) {
    const int64_t n = (int64_t)h * w * l;
    if (gbias)
        for (int co = 0; co < oc; ++co) {
            float s = 0.0f;
            for (int64_t i = 0; i < n; ++i) s += gout[(int64_t)co * n + i];
            gbias[co] += s;
        }
    for (int co = 0; co < oc; ++co)
        for (int ci = 0; ci < ic; ++ci) {
            const float *go = gout + (int64_t)co * n;
            const float *src = in + (int64_t)ci * n;
            for (int t = 0; t < 27; ++t) {
                const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
                const int64_t ki = ((int64_t)co * ic + ci) * 27 + t;
                if (gk) {
                    float s = 0.0f;
                    for (int z = 0; z < l; ++z) {
                        if (z + dz < 0 || z + dz >= l) continue;
                        for (int y = 0; y < w; ++y) {
                            if (y + dy < 0 || y + dy >= w) continue;
                            for (int x = 0; x < h; ++x) {
                                if (x + dx < 0 || x + dx >= h) continue;
                                s += go[vidx(h, w, x, y, z)] * src[vidx(h, w, x + dx, y + dy, z + dz)];
                            }
                        }
                    }
                    gk[ki] += s;
                }
                if (gin && k[ki] != 0.0f) {
                    float *dst = gin + (int64_t)ci * n;
                    const float kv = k[ki];
                    for (int z = 0; z < l; ++z) {
                        if (z - dz < 0 || z - dz >= l) continue;
                        for (int y = 0; y < w; ++y) {
                            if (y - dy < 0 || y - dy >= w) continue;
                            for (int x = 0; x < h; ++x) {
                                if (x - dx < 0 || x - dx >= h) continue;
                                dst[vidx(h, w, x, y, z)] += kv * go[vidx(h, w, x - dx, y - dy, z - dz)];
                            }
                        }
                    }
                }
            }
        }
}

/* ------------------------------------------------------------ field algebra */

/* field_ops.hpp:42-49 */
void mdo_compose_fwd(const float *prev, const float *res, int h, int w, int l, float *out) {
    const int64_t n = (int64_t)h * w * l;
    mdo_warp_fwd(prev, 3, h, w, l, res, out);
    for (int64_t i = 0; i < 3 * n; ++i) out[i] += res[i];
}

/* tape order of op_compose (ops.hpp:295-298 = op_add(res, op_warp(prev,res))):
 * the add node replays first (tape.hpp:146-156), then warp_bwd. */
void mdo_compose_bwd(const float *prev, const float *res, int h, int w, int l,
                     const float *gout, float *gprev, float *gres) {
    const int64_t n = (int64_t)h * w * l;
    if (gres)
        for (int64_t i = 0; i < 3 * n; ++i) gres[i] += gout[i];
    mdo_warp_bwd(prev, 3, h, w, l, res, gout, gprev, gres);
}

/* reghead.hpp:60-67: phi = v / 2^T, then T self-compositions */
void mdo_scaling_squaring(const float *vel, int h, int w, int l, int steps, float *out) {
    const int64_t n3 = 3 * (int64_t)h * w * l;
    const float inv = 1.0f / (float)(1 << steps);
    for (int64_t i = 0; i < n3; ++i) out[i] = vel[i] * inv;
    /* scratch on the heap: compose reads phi twice while writing */
    float *tmp = (float *)malloc((size_t)n3 * sizeof(float));
    for (int s = 0; s < steps; ++s) {
        mdo_compose_fwd(out, out, h, w, l, tmp);
        for (int64_t i = 0; i < n3; ++i) out[i] = tmp[i];
    }
    free(tmp);
}

/* ---------------------------------------------------------- Q/K projection */

/* ops.hpp:387-413: out[p,k] = b[k] + sum_c W[k,c] * in[c,p], summed in channel
 * order starting from the bias */
void mdo_linear_proj_fwd(const float *in, int c, int64_t n, const float *weight,
                         const float *bias, int K, float *out) {
    for (int64_t p = 0; p < n; ++p)
        for (int k = 0; k < K; ++k) {
            float s = bias[k];
            for (int ch = 0; ch < c; ++ch) s += weight[(int64_t)k * c + ch] * in[ch * n + p];
            out[p * K + k] = s;
        }
}

/* ops.hpp:414-433 (tape closure): per position, per output k with g != 0 */
void mdo_linear_proj_bwd(const float *in, int c, int64_t n, const float *weight, int K,
                         const float *gout, float *gin, float *gw, float *gb) {
    for (int64_t p = 0; p < n; ++p)
        for (int k = 0; k < K; ++k) {
            const float g = gout[p * K + k];
            if (g == 0.0f) continue;
            if (gb) gb[k] += g;
            for (int ch = 0; ch < c; ++ch) {
                if (gw) gw[(int64_t)k * c + ch] += g * in[ch * n + p];
                if (gin) gin[ch * n + p] += g * weight[(int64_t)k * c + ch];
            }
        }
}

/* ops.hpp:445-461: two-pass mean / biased variance, inv = 1/sqrt(var + eps) */
static void ln_stats(const float *src, int K, float eps, float *mean_out, float *inv_out) {
    float mean = 0.0f;
    for (int k = 0; k < K; ++k) mean += src[k];
    mean /= (float)K;
    float var = 0.0f;
    for (int k = 0; k < K; ++k) var += (src[k] - mean) * (src[k] - mean);
    var /= (float)K;
    *mean_out = mean;
    *inv_out = 1.0f / sqrtf(var + eps);
}

void mdo_layer_norm_fwd(const float *in, int64_t n, int K, const float *gamma,
                        const float *beta, float eps, float *out) {
    for (int64_t p = 0; p < n; ++p) {
        const float *src = in + p * K;
        float mean, inv;
        ln_stats(src, K, eps, &mean, &inv);
        for (int k = 0; k < K; ++k) out[p * K + k] = gamma[k] * (src[k] - mean) * inv + beta[k];
    }
}

/* ops.hpp:462-494 */
void mdo_layer_norm_bwd(const float *in, int64_t n, int K, const float *gamma, float eps,
                        const float *gout, float *gin, float *gg, float *gb) {
    for (int64_t p = 0; p < n; ++p) {
        const float *src = in + p * K;
        const float *go = gout + p * K;
        float mean, inv;
        ln_stats(src, K, eps, &mean, &inv);
        float sum_g = 0.0f, sum_gx = 0.0f;
        for (int k = 0; k < K; ++k) {
            const float xh = (src[k] - mean) * inv;
            sum_g += go[k] * gamma[k];
            sum_gx += go[k] * gamma[k] * xh;
        }
        const float mg = sum_g / (float)K;
        const float mgx = sum_gx / (float)K;
        for (int k = 0; k < K; ++k) {
            const float xh = (src[k] - mean) * inv;
            if (gg) gg[k] += go[k] * xh;
            if (gb) gb[k] += go[k];
            if (gin) gin[p * K + k] += inv * (go[k] * gamma[k] - mg - xh * mgx);
        }
    }
}

/* ------------------------------------------------------------- optimizers */

/* engine.hpp:279-298 */
void mdo_adam_step(float *value, const float *grad, float *m, float *v, int64_t n, double lr,
                   double beta1, double beta2, double eps, int64_t t) {
    const double bc1 = 1.0 - pow(beta1, (double)t);
    const double bc2 = 1.0 - pow(beta2, (double)t);
    for (int64_t j = 0; j < n; ++j) {
        const double g = (double)grad[j];
        const double mj = beta1 * (double)m[j] + (1.0 - beta1) * g;
        const double vj = beta2 * (double)v[j] + (1.0 - beta2) * g * g;
        m[j] = (float)mj;
        v[j] = (float)vj;
        const double update = lr * (mj / bc1) / (sqrt(vj / bc2) + eps);
        value[j] = (float)((double)value[j] - update);
    }
}

/* engine.hpp:306-311 */
void mdo_sgd_step(float *value, const float *grad, int64_t n, double lr) {
    for (int64_t j = 0; j < n; ++j) value[j] = (float)((double)value[j] - lr * (double)grad[j]);
}
