/*
 * mdo.h — CPU ORACLE for the ModeT hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This is a plain-C restatement of the reference algorithms (mdreg, the CPU
 * C++20 re-creation of ModeTv2 under /root/reference/proj).  It exists so the
 * tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg can check the
 * CUDA path.  Nothing in the product (paper_2403_16526_b200/, include/) links
 * or calls it.
 *
 * Parity pinning: every function here is checked against
 *   (1) oracle/_ref/libmdreg_ref.so — the reference headers compiled unmodified
 *       from /root/reference/proj/include by oracle/Makefile (bit-exact
 *       comparison, both built with -ffp-contract=off), and
 *   (2) the committed golden fixtures in tests/golden/ (generated from (1) by
 *       tests/golden/make_golden.py) plus the reference's known-answer tests
 *       restated in tests/test_oracle.py.
 *
 * Conventions (reference common.hpp:56-59, volume.hpp:41-80):
 *   dims (h, w, l) = extents along x, y, z; flat index p = (z*w + y)*h + x.
 *   Feature maps / fields are channel-major {C, n}.  Q/K in the reference
 *   attention API are position-major {n, S*d}.
 */
#ifndef MDO_H
#define MDO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* reference rng.hpp:23-67 — splitmix64 with Box-Muller normal (one cached). */
typedef struct {
    uint64_t state;
    int has_spare;
    double spare;
} mdo_rng;

void mdo_rng_init(mdo_rng *r, uint64_t seed);
uint64_t mdo_rng_next_u64(mdo_rng *r);
double mdo_rng_uniform01(mdo_rng *r);
double mdo_rng_uniform(mdo_rng *r, double lo, double hi);
int mdo_rng_uniform_int(mdo_rng *r, int lo, int hi);
double mdo_rng_normal(mdo_rng *r);
/* float fills, consuming the stream in element order */
void mdo_rng_fill_uniform(mdo_rng *r, float *out, int64_t n, double lo, double hi);
void mdo_rng_fill_normal(mdo_rng *r, float *out, int64_t n, double mean, double sd);

/* attention.hpp:57-60 */
void mdo_window_offset(int o, int nb, int off[3]);

/* attention.hpp:83-123.  Returns 0, or 1 on a non-finite logit with the first
 * offending (x,y,z,head) in loop order written to bad[4] (may be NULL). */
int mdo_na_fwd(const float *Q, const float *K, const float *B, int h, int w, int l, int S,
               int hd, int nb, float *W, int bad[4]);
/* attention.hpp:127-166 (accumulates into gQ, gK, gB) */
void mdo_na_bwd(const float *Q, const float *K, const float *W, int h, int w, int l, int S,
                int hd, int nb, const float *gW, float *gQ, float *gK, float *gB);
/* attention.hpp:282-298 */
void mdo_subfields_fwd(const float *W, int h, int w, int l, int S, int nb, float *out);
/* attention.hpp:301-316 (accumulates into gW) */
void mdo_subfields_bwd(int h, int w, int l, int S, int nb, const float *gout, float *gW);
/* attention.hpp:421-427: 1 if every row sums to 1 within tol */
int mdo_rows_normalized(const float *W, int64_t rows, int win, double tol);

/* sampling.hpp:38-49 */
void mdo_resolve_axis(float x, int dim, int *i0, int *i1, float *f, int *live);
/* sampling.hpp:123-135 */
void mdo_warp_fwd(const float *in, int C, int h, int w, int l, const float *field, float *out);
/* sampling.hpp:139-167 (accumulates; gin / gfield may be NULL) */
void mdo_warp_bwd(const float *in, int C, int h, int w, int l, const float *field,
                  const float *gout, float *gin, float *gfield);
/* sampling.hpp:225-242 */
void mdo_upsample2_fwd(const float *in, int C, int h, int w, int l, int th, int tw, int tl,
                       float scale, float *out);
/* sampling.hpp:245-262 (accumulates) */
void mdo_upsample2_bwd(int C, int h, int w, int l, int th, int tw, int tl, float scale,
                       const float *gout, float *gin);
/* sampling.hpp:266-271: 1 if target within the doubling range */
int mdo_upsample_target_ok(int h, int w, int l, int th, int tw, int tl);

/* ops.hpp:58-74 (kernel layout [oc][ic][dz][dy][dx]; bias may be NULL) */
void mdo_conv3_fwd(const float *in, int ic, int h, int w, int l, const float *k,
                   const float *bias, int oc, float *out);
/* ops.hpp:77-99 (accumulates; gin, gk, gbias may be NULL) */
void mdo_conv3_bwd(const float *in, int ic, int h, int w, int l, const float *k, int oc,
                   const float *gout, float *gin, float *gk, float *gbias);

/* field_ops.hpp:42-49 / ops.hpp:295-298: out = res + warp(prev, res) */
void mdo_compose_fwd(const float *prev, const float *res, int h, int w, int l, float *out);
/* backward of compose (accumulates into gprev, gres; either may be NULL) */
void mdo_compose_bwd(const float *prev, const float *res, int h, int w, int l,
                     const float *gout, float *gprev, float *gres);
/* reghead.hpp:60-67 (plain scaling and squaring) */
void mdo_scaling_squaring(const float *vel, int h, int w, int l, int steps, float *out);

/* engine.hpp:268-298 AdamOptimizer::step for one parameter tensor (double
 * arithmetic per element, float storage); t = step count after increment */
void mdo_adam_step(float *value, const float *grad, float *m, float *v, int64_t n, double lr,
                   double beta1, double beta2, double eps, int64_t t);
/* engine.hpp:306-311 sgd_step */
void mdo_sgd_step(float *value, const float *grad, int64_t n, double lr);

/* ops.hpp:387-413 op_linear_proj forward: in {c, n} channel-major, weight
 * {K, c}, bias {K} -> out position-major {n, K} */
void mdo_linear_proj_fwd(const float *in, int c, int64_t n, const float *weight,
                         const float *bias, int K, float *out);
/* ops.hpp:414-433 backward (accumulates; gin/gw/gb may be NULL; g == 0 skipped) */
void mdo_linear_proj_bwd(const float *in, int c, int64_t n, const float *weight, int K,
                         const float *gout, float *gin, float *gw, float *gb);
/* ops.hpp:439-461 op_layer_norm forward over the trailing K axis of {n, K} */
void mdo_layer_norm_fwd(const float *in, int64_t n, int K, const float *gamma,
                        const float *beta, float eps, float *out);
/* ops.hpp:462-494 backward (accumulates; gin/gg/gb may be NULL) */
void mdo_layer_norm_bwd(const float *in, int64_t n, int K, const float *gamma, float eps,
                        const float *gout, float *gin, float *gg, float *gb);

#ifdef __cplusplus
}
#endif
#endif
