/*
 * mdg.h — C ABI of the B200-native ModeT hot path (sm_100a).
 *
 * Drop-in boundary for the mdreg reference (/root/reference/proj).  Two tiers:
 *
 *  1. Reference-shaped kernel tier ("mdg_na_*", "mdg_subfields_*", "mdg_warp_*",
 *     "mdg_upsample2_*", "mdg_conv3_*", "mdg_compose_*"): one entry point per
 *     `mdreg::kern::` function on the path, same argument meaning, same
 *     layouts, same overwrite/accumulate rules.  Each cites the reference
 *     function it replaces (paths relative to proj/include/mdreg/).
 *  2. Fused tier ("mdg_modet_*"): the B200-native ModeT operator.  Q·K over
 *     the nb^3 window -> softmax -> sum of offsets in one kernel; the nb^3
 *     weight tensor W is never materialised (optional output for parity).
 *     The backward recomputes W from (Q, K, B, LSE) and fuses dQ, dK (gather,
 *     no atomics) and dB (deterministic two-stage reduction).
 *
 * Conventions (reference common.hpp:40-74, volume.hpp:26-94):
 *  - dims {h, w, l} = extents along x, y, z; voxel p = (z*w + y)*h + x.
 *  - Feature maps and fields are channel-major {C, n}; fields have C = 3
 *    (x, y, z components, voxel units of their own grid).
 *  - All values fp32; all sizes int32 (n = h*w*l < 2^31).
 *  - Device-pointer entry points take a cudaStream_t as `void *stream`
 *    (NULL = legacy default stream) and are stream-ordered: they return once
 *    the work is enqueued.  `*_host` entry points take host pointers and are
 *    synchronous, exactly like the reference's CPU functions.
 *  - Forward entry points OVERWRITE their outputs.  Backward entry points
 *    ACCUMULATE (+=) into their gradient outputs, as the reference does
 *    (attention.hpp:153-161, sampling.hpp:153-164, ops.hpp:84-96); a NULL
 *    gradient pointer skips that gradient.
 *
 * Errors: every entry point returns an mdg_status.  A C ABI cannot throw, so
 * the reference's exceptions map to codes and a per-thread message:
 *    invalid_input  -> MDG_EINVAL   (shape / config / range violations)
 *    numeric_error  -> MDG_ENUMERIC (non-finite attention logit)
 *    CUDA failures  -> MDG_ECUDA
 * Non-finite logits are detected on the device; the first offending
 * (x, y, z, head) in the reference's loop order (head-major, then z, y, x) is
 * recorded.  The reference-shaped tier and the *_host calls check it before
 * returning (they synchronise the stream), exactly reproducing the
 * reference's throw; the fused tier defers the check to
 * mdg_check_numeric(stream) so a pyramid step stays asynchronous.
 */
#ifndef MDG_H
#define MDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MDG_OK = 0,
    MDG_EINVAL = 1,
    MDG_ENUMERIC = 2,
    MDG_ECUDA = 3,
    MDG_EPARSE = 4 /* parse_error: malformed or truncated files (common.hpp:29-32) */
} mdg_status;

/* Q/K layouts accepted by the fused tier. */
typedef enum {
    MDG_QK_POSMAJOR = 0, /* reference layout {n, S*d} (attention.hpp:77-78) */
    MDG_QK_PLANAR = 1    /* native layout {S*d, n}: one coalesced plane per channel */
} mdg_qk_layout;

typedef struct {
    int h, w, l;
} mdg_dims3;

/* ------------------------------------------------------------- diagnostics */
const char *mdg_last_error(void);
/* position of the last non-finite logit reported by MDG_ENUMERIC */
void mdg_last_error_position(int *x, int *y, int *z, int *head);
/* 1 if the library was built for and runs on an sm_100a device */
int mdg_device_ok(void);
const char *mdg_build_info(void);
/* synchronise `stream` and return MDG_ENUMERIC if any fused-tier kernel on
 * this device recorded a non-finite logit since the last check; the position
 * is decoded against `d`, the dims of the attention call being checked */
mdg_status mdg_check_numeric(mdg_dims3 d, void *stream);
/* number of kernels this library launched since load (host-side counter) */
int64_t mdg_launch_count(void);
/* Deterministic mode (process-wide; initial value from the environment
 * variable MDG_DETERMINISTIC).  Off: the warp / compose input gradients are
 * scattered with float atomics (fastest; the summation order at a shared
 * corner varies between runs).  On: whole-volume calls scatter into a 64-bit
 * fixed-point accumulator (integer adds: order independent; ~1.7x the warp
 * backward's time and 8 bytes of pool scratch per gin element), voxel-range
 * calls gather per target in a fixed order (~3x), so every result — and a
 * whole pairwise optimisation — is bit-identical from run to run, as the
 * reference guarantees (test_engine.cpp:194-213).  Every other
 * kernel is deterministic in both modes.  Returns the previous setting. */
int mdg_set_deterministic(int on);
int mdg_get_deterministic(void);

/* ---------------------------------------------------- index logic (exact) */
/* attention.hpp:57-60 window_offset: slot o -> (dx, dy, dz), x fastest */
mdg_status mdg_window_offset(int o, int nb, int off[3]);
/* sampling.hpp:38-49 resolve_axis evaluated ON THE DEVICE for n coordinates
 * (used to prove the integer corner logic is bit-exact) */
mdg_status mdg_resolve_axis(const float *x, int n, int dim, int *i0, int *i1, float *f,
                            int *live, void *stream);

/* ====================== reference-shaped kernel tier ====================== */

/* attention.hpp:83-123 kern::na_fused_fwd.  Q, K {n, S*hd} position-major;
 * B {S, nb^3}; W {S, n, nb^3} (overwritten). */
mdg_status mdg_na_fused_fwd(const float *Q, const float *K, const float *B, mdg_dims3 d,
                            int S, int hd, int nb, float *W, void *stream);
/* attention.hpp:127-166 kern::na_fused_bwd (accumulates gQ, gK, gB) */
mdg_status mdg_na_fused_bwd(const float *Q, const float *K, const float *W, mdg_dims3 d,
                            int S, int hd, int nb, const float *gW, float *gQ, float *gK,
                            float *gB, void *stream);
/* attention.hpp:282-298 kern::subfields_fwd: W {S,n,nb^3} -> out {3S, n} */
mdg_status mdg_subfields_fwd(const float *W, mdg_dims3 d, int S, int nb, float *out,
                             void *stream);
/* attention.hpp:301-316 kern::subfields_bwd (accumulates gW) */
mdg_status mdg_subfields_bwd(mdg_dims3 d, int S, int nb, const float *gout, float *gW,
                             void *stream);
/* attention.hpp:421-427 (op_subfields row check): MDG_EINVAL if some row of W
 * does not sum to 1 within tol */
mdg_status mdg_subfields_check_rows(const float *W, mdg_dims3 d, int S, int nb, float tol,
                                    void *stream);

/* sampling.hpp:123-135 kern::warp_fwd: out_c(x) = in_c(x + field(x)) */
mdg_status mdg_warp_fwd(const float *in, int C, mdg_dims3 d, const float *field, float *out,
                        void *stream);
/* sampling.hpp:139-167 kern::warp_bwd (accumulates; gin/gfield nullable) */
mdg_status mdg_warp_bwd(const float *in, int C, mdg_dims3 d, const float *field,
                        const float *gout, float *gin, float *gfield, void *stream);
/* the same two calls over the voxel range [pb, pe) only (arrays full-size,
 * global coordinates): a z-slab's share (depth-slab decomposition) or a
 * pipeline chunk.  Bit-identical per voxel to the whole-volume calls. */
mdg_status mdg_warp_fwd_range(const float *in, int C, mdg_dims3 d, const float *field,
                              float *out, int64_t pb, int64_t pe, void *stream);
mdg_status mdg_warp_bwd_range(const float *in, int C, mdg_dims3 d, const float *field,
                              const float *gout, float *gin, float *gfield, int64_t pb,
                              int64_t pe, void *stream);
/* Depth-slab warp (the per-rank call of a z-decomposed
 * kern::warp_fwd / warp_bwd, sampling.hpp:123 / 139): the voxels of planes
 * [z0, z1) of a volume of dims d.  in / gin hold only the planes [zi0, zi1)
 * (the slab plus the field's reach), field / out / gout / gfield only the
 * planes [z0, z1); results equal mdg_warp_*_range over full-size buffers.
 * A field that samples outside [zi0, zi1) -> MDG_EINVAL (checked on the
 * device, reported synchronously).  gin accumulates by fp32 atomics. */
mdg_status mdg_warp_fwd_slab(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                             const float *field, float *out, int z0, int z1, void *stream);
mdg_status mdg_warp_bwd_slab(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                             const float *field, const float *gout, float *gin, float *gfield,
                             int z0, int z1, void *stream);
/* The same without the synchronous window check: a violation ORs 1 into the
 * caller's device word *err (read it when convenient; graph-capturable). */
mdg_status mdg_warp_fwd_slab_async(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                                   const float *field, float *out, int z0, int z1,
                                   unsigned *err, void *stream);
mdg_status mdg_warp_bwd_slab_async(const float *in, int C, mdg_dims3 d, int zi0, int zi1,
                                   const float *field, const float *gout, float *gin,
                                   float *gfield, int z0, int z1, unsigned *err, void *stream);
/* sampling.hpp:225-242 kern::upsample2_fwd (target range checked as in
 * sampling.hpp:266-271 -> MDG_EINVAL) */
mdg_status mdg_upsample2_fwd(const float *in, int C, mdg_dims3 d, mdg_dims3 td, float scale,
                             float *out, void *stream);
/* sampling.hpp:245-262 kern::upsample2_bwd (accumulates gin) */
mdg_status mdg_upsample2_bwd(int C, mdg_dims3 d, mdg_dims3 td, float scale, const float *gout,
                             float *gin, void *stream);
/* ops.hpp:58-74 kern::conv3_fwd (zero-padded 3x3x3 correlation, kernel
 * [oc][ic][dz][dy][dx]; bias nullable).  RegHead fusion (reghead.hpp:42-47)
 * is this with ic = 3S, oc = 3. */
mdg_status mdg_conv3_fwd(const float *in, int ic, mdg_dims3 d, const float *k,
                         const float *bias, int oc, float *out, void *stream);
/* ops.hpp:77-99 kern::conv3_bwd (accumulates; gin/gk/gbias nullable) */
mdg_status mdg_conv3_bwd(const float *in, int ic, mdg_dims3 d, const float *k, int oc,
                         const float *gout, float *gin, float *gk, float *gbias, void *stream);
/* field_ops.hpp:42-49 / ops.hpp:295-298: out = res + warp(prev, res) */
mdg_status mdg_compose_fwd(const float *prev, const float *res, mdg_dims3 d, float *out,
                           void *stream);
/* backward of op_compose (accumulates gprev, gres; nullable) */
mdg_status mdg_compose_bwd(const float *prev, const float *res, mdg_dims3 d,
                           const float *gout, float *gprev, float *gres, void *stream);
/* reghead.hpp:52-67 scaling and squaring: out = (v/2^T) composed T times.
 * `saved` (nullable, (steps+1)*3n floats) receives the intermediate fields
 * phi_0 .. phi_T that mdg_scaling_squaring_bwd needs. */
mdg_status mdg_scaling_squaring_fwd(const float *vel, mdg_dims3 d, int steps, float *out,
                                    float *saved, void *stream);
/* backward of op_scaling_squaring given `saved` from the forward
 * (accumulates gvel) */
mdg_status mdg_scaling_squaring_bwd(const float *saved, mdg_dims3 d, int steps,
                                    const float *gout, float *gvel, void *stream);

/* ============================== fused tier ============================== */

/* ModeT forward.  Q, K in `layout`; B {S, nb^3}.  Outputs:
 *   SF  {3S, n} sub-flows (what kern::subfields_fwd(na_fused_fwd(..)) gives)
 *   LSE {S, n}  per-row log-sum-exp, saved for the backward
 *   W   {S, n, nb^3} nullable — materialised only for parity checks. */
mdg_status mdg_modet_fwd(const float *Q, const float *K, const float *B, mdg_dims3 d, int S,
                         int hd, int nb, int layout, float *SF, float *LSE, float *W,
                         void *stream);
/* ModeT backward.  Given the forward's SF and LSE and the upstream gradient
 * gSF {3S, n}, produces gQ, gK (same layout as Q, K) and gB {S, nb^3}.
 * Equivalent to subfields_bwd + na_fused_bwd of the reference.
 * accumulate != 0: gQ/gK/gB += (the reference rule); accumulate == 0: gQ and
 * gK are overwritten (saves their read-modify-write; gB always accumulates). */
mdg_status mdg_modet_bwd(const float *Q, const float *K, const float *B, const float *SF,
                         const float *LSE, const float *gSF, mdg_dims3 d, int S, int hd, int nb,
                         int layout, float *gQ, float *gK, float *gB, int accumulate,
                         void *stream);

/* Q/K projection (attention.hpp:351-356 op_project_qk = op_layer_norm(
 * op_linear_proj(.)) ops.hpp:387-497, shared weights, LN eps 1e-5 over all
 * K = S*hd outputs of a voxel).  f, m {C, n} channel-major; weight {K, C};
 * bias, ln_g, ln_b {K}.  Q, K written in `layout` (MDG_QK_POSMAJOR = the
 * reference {n, K}; MDG_QK_PLANAR = {K, n}, what the fused tier reads).  m/K
 * may both be NULL to project one input. */
mdg_status mdg_project_qk_fwd(const float *f, const float *m, int C, int64_t n,
                              const float *weight, const float *bias, const float *ln_g,
                              const float *ln_b, int K, int layout, float *Q, float *Kout,
                              void *stream);
/* backward (ops.hpp:414-433, 462-494): accumulates gf, gm {C, n} and the
 * parameter gradients; every output pointer nullable; K <= 64 */
mdg_status mdg_project_qk_bwd(const float *f, const float *m, int C, int64_t n,
                              const float *weight, const float *bias, const float *ln_g, int K,
                              int layout, const float *gQ, const float *gK, float *gf,
                              float *gm, float *gweight, float *gbias, float *gln_g,
                              float *gln_b, void *stream);

/* ===================== registration objective (§8f) =====================
 * op_total_loss (objective.hpp:71-78): warped = warp(moving, phi);
 *   total = NCC(fixed, warped; window) + lambda * grad_reg(phi)
 * (op_ncc_loss objective.hpp:39-69, op_grad_reg ops.hpp:326-382).  fixed,
 * moving: single-channel volumes {n}; phi {3, n}.  `terms` (device, 3 floats)
 * receives {total, ncc, reg}; `warped` (nullable) the warped moving image. */
mdg_status mdg_total_loss_fwd(const float *fixed, const float *moving, const float *phi,
                              mdg_dims3 d, int window, float lambda, float *terms,
                              float *warped, void *stream);
/* backward of `seed * total`: accumulates gphi {3, n} and gmoving {n}
 * (each nullable) */
mdg_status mdg_total_loss_bwd(const float *fixed, const float *moving, const float *phi,
                              mdg_dims3 d, int window, float lambda, float seed, float *gphi,
                              float *gmoving, void *stream);

/* ============================ optimizers (§8f) ===========================
 * engine.hpp:268-298 AdamOptimizer::step on one parameter tensor: value, m, v
 * updated in place from grad; t = the step count after increment (1-based).
 * Per-element arithmetic in double as the reference (bit-identical). */
mdg_status mdg_adam_step(float *value, const float *grad, float *m, float *v, int64_t n,
                         double lr, double beta1, double beta2, double eps, int64_t t,
                         void *stream);
/* engine.hpp:306-311 sgd_step */
mdg_status mdg_sgd_step(float *value, const float *grad, int64_t n, double lr, void *stream);

/* ========================= label evaluation (§8f) ========================
 * metrics.cpp:145-164 warp_labels: nearest-neighbour pull of int32 labels by
 * phi {3, n} (floor(x + phi + 0.5f), clamped) — bit-identical */
mdg_status mdg_warp_labels(const int *labels, mdg_dims3 d, const float *phi, int *out,
                           void *stream);
/* metrics.cpp:100-129 mean_dice over the labels present in a or b (label 0
 * excluded); labels must lie in [0, max_label].  Synchronous (the result is a
 * host double); bit-identical to the reference. */
mdg_status mdg_mean_dice(const int *a, const int *b, int64_t n, int max_label, double *dice,
                         void *stream);

/* ============================ encoder (§8f) ===============================
 * op_encode (encoder.hpp:102-116): five shared-weight conv blocks
 * (conv3 -> InstanceNorm -> LeakyReLU, twice; encoder.hpp:87-91) with 2x
 * average pooling between levels (sampling.hpp:171-219).  Channels at level L
 * are base << (L-1).  The object owns the saved activations of one image. */
typedef struct {
    const float *w1, *b1, *g1, *be1; /* conv1 {C,Cin,3,3,3}, {C}; norm1 gamma/beta {C} */
    const float *w2, *b2, *g2, *be2; /* conv2 {C,C,3,3,3}, ... */
} mdg_block_params;
typedef struct {
    float *w1, *b1, *g1, *be1, *w2, *b2, *g2, *be2; /* accumulated; nullable */
} mdg_block_grads;
/* The encoder's conv3 on its own (op_conv3d ops.hpp:137-238, any channel
 * counts): out {oc, n} = conv(in {ic, n}, w {oc, ic, 3,3,3}) + b.  FMA-
 * contracted fp32 (relative-norm parity, not bit-exact: the bit-exact
 * reference-order kernel is mdg_conv3_fwd).  Backward ACCUMULATES gin, gw, gb
 * (each nullable). */
mdg_status mdg_encoder_conv3_fwd(const float *in, int ic, mdg_dims3 d, const float *w,
                                 const float *b, int oc, float *out, void *stream);
mdg_status mdg_encoder_conv3_bwd(const float *in, int ic, mdg_dims3 d, const float *w, int oc,
                                 const float *gout, float *gin, float *gw, float *gb,
                                 void *stream);
/* NCC of one depth slab (op_ncc_loss objective.hpp:39-69 split along z):
 * fixed / warped {1, l, w, h} on the slab's EXTENDED grid e = its own planes
 * plus window/2 halo planes per side (zero beyond the volume); the planes
 * [zv0, zv1) of e lie inside the volume (the window counts).
 *   fwd: *cc_sum (device) = sum of cc over the slab's own planes
 *        [window/2, e.l - window/2); the caller all-reduces it, ncc = -sum/N
 *   bwd: gwarped {e} (written) = d(gcc * sum cc)/dwarped; its halo planes hold
 *        the contributions that belong to the neighbours */
mdg_status mdg_ncc_slab_fwd(const float *fixed, const float *warped, mdg_dims3 e, int window,
                            int zv0, int zv1, float *cc_sum, void *stream);
mdg_status mdg_ncc_slab_bwd(const float *fixed, const float *warped, mdg_dims3 e, int window,
                            int zv0, int zv1, float gcc, float *gwarped, void *stream);
/* as mdg_ncc_slab_bwd with dL/dcc = gcc * (*gscale), gscale a device scalar
 * (the upstream gradient without a host round trip: graph-capturable) */
mdg_status mdg_ncc_slab_bwd_dev(const float *fixed, const float *warped, mdg_dims3 e, int window,
                                int zv0, int zv1, float gcc, const float *gscale,
                                float *gwarped, void *stream);
/* Depth-slab instance norm + leaky ReLU: op_instance_norm (ops.hpp:162-221)
 * and op_leaky_relu (:224-238) split at their two global reductions, so a
 * slab-decomposed caller all-reduces the per-channel sums in between.
 * x {C, n} (this slab's voxels).
 *   mdg_in_slab_sums: sums[c] = sum x (mean NULL) or sum (x - mean[c])^2 (fp64)
 *   mdg_in_lrelu_apply: z = lrelu(g (x - mean) inv + b), given the global
 *     mean and inv = 1/sqrt(var + 1e-5)
 *   mdg_in_lrelu_bwd_sums: sums {C, 2} = {sum gy, sum gy xh} (gy = gz lrelu', fp64)
 *     over the slab — also the beta / gamma gradients before the all-reduce
 *   mdg_in_lrelu_bwd_apply: gx (written) from the all-reduced sums over the
 *     nstat voxels of the whole volume (ops.hpp:206-212) */
mdg_status mdg_in_slab_sums(const float *x, int C, int64_t n, const float *mean, double *sums,
                            void *stream);
mdg_status mdg_in_lrelu_apply(const float *x, int C, int64_t n, const float *mean,
                              const float *inv, const float *g, const float *b, float slope,
                              float *z, void *stream);
mdg_status mdg_in_lrelu_bwd_sums(const float *x, const float *gz, int C, int64_t n,
                                 const float *mean, const float *inv, const float *g,
                                 const float *b, float slope, double *sums, void *stream);
mdg_status mdg_in_lrelu_bwd_apply(const float *x, const float *gz, int C, int64_t n,
                                  const float *mean, const float *inv, const float *g,
                                  const float *b, float slope, const float *sums, int64_t nstat,
                                  float *gx, void *stream);
/* sampling.hpp:171-219 kern::avg_pool_fwd / avg_pool_bwd (2x, odd extents
 * repeat their last voxel; the backward accumulates gin) */
mdg_status mdg_avgpool2_fwd(const float *in, int C, mdg_dims3 d, float *out, void *stream);
mdg_status mdg_avgpool2_bwd(const float *gout, int C, mdg_dims3 d, float *gin, void *stream);
typedef struct mdg_encoder mdg_encoder;
/* dims of the full-resolution image (>= 16 per axis, encoder.hpp:95-99) */
mdg_status mdg_encoder_create(mdg_dims3 d, int base_channels, int levels, float slope,
                              mdg_encoder **out);
void mdg_encoder_destroy(mdg_encoder *e);
/* image {1, n}; params[levels]; features[L] {C_L, n_L}, fine -> coarse
 * (op_encode's order) */
mdg_status mdg_encoder_forward(mdg_encoder *e, const float *image,
                               const mdg_block_params *params, float *const *features,
                               void *stream);
/* backward of the last forward: gfeatures[L] (entries nullable) -> param
 * grads (accumulated) and gimage (accumulated, nullable) */
mdg_status mdg_encoder_backward(mdg_encoder *e, const float *const *gfeatures,
                                const mdg_block_grads *grads, float *gimage, void *stream);

/* ========================== whole model (§8f) =============================
 * ModelParams of ModelConfig::small_preset (engine.hpp:38-44, 114-140) and
 * one run_loss_step (engine.hpp:316-340) / Adam update (engine.hpp:389-398)
 * as one native object: encoder x2 -> decoding pyramid -> total loss, the
 * backward into the 75 parameter gradients, and AdamOptimizer::step.  The
 * 75 tensors follow ModelParams::all_tensors (engine.hpp:121-133). */
typedef struct mdg_model mdg_model;
/* number of parameter tensors (75) and, if `sizes` is non-NULL, the element
 * count of each; returns the total element count */
int64_t mdg_model_param_count(int *ntensors, int64_t *sizes);
/* init_model(small_preset, seed) (engine.hpp:143-166) into HOST buffers
 * params_host[75] — bit-identical to the reference's Rng draws */
mdg_status mdg_model_init(uint64_t seed, float *const *params_host);
/* params[75]: DEVICE tensors, caller-owned, updated in place by adam_step.
 * lambda / ncc_window: LossConfig (objective.hpp:21-31).  check_finite: as
 * mdg_pyramid_config::check_finite. */
mdg_status mdg_model_create(mdg_dims3 d, float *const *params, float lambda, int ncc_window,
                            int check_finite, mdg_model **out);
void mdg_model_destroy(mdg_model *m);
/* the 75 device gradient tensors (valid until destroy) */
float *const *mdg_model_grads(mdg_model *m);
/* fixed, moving: device {n}.  terms (device, 3 floats, nullable) <- {total,
 * ncc, reg}; phi (device {3, n}, nullable) <- the field.  backward != 0 also
 * zeroes and fills the gradients. */
mdg_status mdg_model_loss_step(mdg_model *m, const float *fixed, const float *moving,
                               int backward, float *terms, float *phi, void *stream);
/* AdamOptimizer::step (engine.hpp:268-298; beta 0.9/0.999, eps 1e-8) over all
 * 75 tensors with the gradients of the last backward */
mdg_status mdg_model_adam_step(mdg_model *m, double lr, void *stream);
/* one PO iteration, loss_step(backward) + adam_step, launched as a CUDA graph
 * captured on the first call and replayed while fixed/moving/terms/lr/stream
 * stay the same (re-captured otherwise) */
mdg_status mdg_model_po_step(mdg_model *m, const float *fixed, const float *moving, double lr,
                             float *terms, void *stream);
/* the model's field {3, n} of the last loss step (device; valid until the next) */
const float *mdg_model_phi(const mdg_model *m);

/* ======================== decoding pyramid driver ========================
 * The decoder half of build_pipeline (engine.hpp:179-219) on device-resident
 * encoder features: per level k (coarse -> fine)
 *     phi_up = upsample_field_2x(phi)          (k > 0, ops.hpp:258)
 *     m_in   = warp(m_k, phi_up)               (k > 0, ops.hpp:275)
 *     Q, K   = project_qk(f_k, m_in)           (attention.hpp:351)
 *     SF     = ModeT(Q, K, rel_bias)           (fused tier)
 *     res    = reghead conv3(SF)               (reghead.hpp:42)
 *     res    = scaling_squaring(res)           (if diffeomorphic, reghead.hpp:52)
 *     phi    = k == 0 ? res : compose(phi_up, res)   (ops.hpp:295)
 * The object owns the saved activations; backward replays the levels in
 * reverse (the tape order of engine.hpp) and ACCUMULATES into the parameter
 * and feature gradients. */
#define MDG_MAX_LEVELS 8
typedef struct {
    int levels;                         /* EncoderConfig::levels (<= MDG_MAX_LEVELS) */
    int heads[MDG_MAX_LEVELS];          /* ModelConfig::heads_per_level, coarse -> fine */
    int channels[MDG_MAX_LEVELS];       /* feature channels per level, coarse -> fine */
    mdg_dims3 dims[MDG_MAX_LEVELS];     /* level grids, coarse -> fine */
    int head_dim;                       /* ModelConfig::head_dim */
    int neighborhood;                   /* must be 3 on the fused tier */
    int diffeomorphic;                  /* ModelConfig::diffeomorphic */
    int ss_steps;                       /* ModelConfig::ss_steps */
    int check_finite;                   /* !=0: forward syncs and raises the non-finite
                                           logit error (attention.hpp:110-114); backward
                                           raises on a non-finite gradient
                                           (tape.hpp:116-120) */
} mdg_pyramid_config;

/* LevelParams (engine.hpp:108-112), device pointers */
typedef struct {
    const float *proj_w;   /* {S*hd, C} */
    const float *proj_b;   /* {S*hd} */
    const float *ln_g;     /* {S*hd} */
    const float *ln_b;     /* {S*hd} */
    const float *rel_bias; /* {S, nb^3} */
    const float *rh_w;     /* {3, 3S, 3, 3, 3} */
    const float *rh_b;     /* {3} */
} mdg_level_params;

/* gradients of LevelParams (accumulated; each pointer nullable) */
typedef struct {
    float *proj_w, *proj_b, *ln_g, *ln_b, *rel_bias, *rh_w, *rh_b;
} mdg_level_grads;

typedef struct mdg_pyramid mdg_pyramid;

/* validates the config (ModelConfig::validate engine.hpp:64-78, level dims
 * must chain by check_upsample_target) and allocates the saved activations */
mdg_status mdg_pyramid_create(const mdg_pyramid_config *cfg, mdg_pyramid **out);
void mdg_pyramid_destroy(mdg_pyramid *p);
/* f_feats[k], m_feats[k]: {C_k, n_k}; params[k]; writes phi {3, n_fine} and,
 * if `residuals` and residuals[k] are non-NULL, each level's residual. */
mdg_status mdg_pyramid_forward(mdg_pyramid *p, const float *const *f_feats,
                               const float *const *m_feats, const mdg_level_params *params,
                               float *phi, float *const *residuals, void *stream);
/* backward of the last forward with dloss/dphi = gphi {3, n_fine}.  grads
 * (array of `levels`, nullable), gf / gm (arrays of `levels` feature-gradient
 * pointers, nullable, entries nullable) accumulate. */
mdg_status mdg_pyramid_backward(mdg_pyramid *p, const float *gphi, const mdg_level_grads *grads,
                                float *const *gf, float *const *gm, void *stream);
/* bytes of device memory the pyramid object holds */
int64_t mdg_pyramid_bytes(const mdg_pyramid *p);

/* layout adapters between the reference {n, C} and native {C, n} */
mdg_status mdg_qk_posmajor_to_planar(const float *src, int64_t n, int C, float *dst,
                                     void *stream);
mdg_status mdg_qk_planar_to_posmajor(const float *src, int64_t n, int C, float *dst,
                                     void *stream);

/* ============================ host-buffer calls ============================
 * Synchronous drop-ins for the reference CPU functions: host pointers in and
 * out; device staging and the copies happen inside the call. */
mdg_status mdg_na_fused_fwd_host(const float *Q, const float *K, const float *B, mdg_dims3 d,
                                 int S, int hd, int nb, float *W);
/* the other reference kern:: functions on host buffers (same semantics as the
 * device calls above: outputs overwritten, gradients accumulated) — what
 * integration/mdreg_b200.hpp binds kern::*<float> to */
mdg_status mdg_na_fused_bwd_host(const float *Q, const float *K, const float *W, mdg_dims3 d,
                                 int S, int hd, int nb, const float *gW, float *gQ, float *gK,
                                 float *gB);
mdg_status mdg_subfields_fwd_host(const float *W, mdg_dims3 d, int S, int nb, float *out);
mdg_status mdg_subfields_bwd_host(mdg_dims3 d, int S, int nb, const float *gout, float *gW);
mdg_status mdg_upsample2_fwd_host(const float *in, int C, mdg_dims3 d, mdg_dims3 td,
                                  float scale, float *out);
mdg_status mdg_upsample2_bwd_host(int C, mdg_dims3 d, mdg_dims3 td, float scale,
                                  const float *gout, float *gin);
mdg_status mdg_conv3_fwd_host(const float *in, int ic, mdg_dims3 d, const float *k,
                              const float *bias, int oc, float *out);
mdg_status mdg_conv3_bwd_host(const float *in, int ic, mdg_dims3 d, const float *k, int oc,
                              const float *gout, float *gin, float *gk, float *gbias);
mdg_status mdg_modet_fwd_host(const float *Q, const float *K, const float *B, mdg_dims3 d,
                              int S, int hd, int nb, int layout, float *SF, float *LSE);
/* accumulate: as mdg_modet_bwd (1: gQ/gK/gB +=, the reference's rule;
 * 0: overwritten, e.g. for a tape's zero-initialised gradients) */
mdg_status mdg_modet_bwd_host(const float *Q, const float *K, const float *B, const float *SF,
                              const float *LSE, const float *gSF, mdg_dims3 d, int S, int hd,
                              int nb, int layout, float *gQ, float *gK, float *gB,
                              int accumulate);
mdg_status mdg_warp_fwd_host(const float *in, int C, mdg_dims3 d, const float *field,
                             float *out);
mdg_status mdg_warp_bwd_host(const float *in, int C, mdg_dims3 d, const float *field,
                             const float *gout, float *gin, float *gfield);

/* ========================= synthetic input streams =========================
 * Bit-identical to the reference's splitmix64/Box-Muller Rng (rng.hpp:23-67),
 * so the GPU and the CPU reference consume identical bytes. */
typedef struct mdg_rng mdg_rng;
mdg_rng *mdg_rng_new(uint64_t seed);
void mdg_rng_free(mdg_rng *r);
void mdg_rng_fill_uniform(mdg_rng *r, float *out, int64_t n, double lo, double hi);
void mdg_rng_fill_normal(mdg_rng *r, float *out, int64_t n, double mean, double sd);
/* synth.cpp:75-90 make_smooth_velocity(dims, seed, magnitude, sigma): host
 * {3, n}, bit-identical to the reference */
mdg_status mdg_synth_smooth_velocity(mdg_dims3 d, uint64_t seed, float magnitude, float sigma,
                                     float *out);
/* tests/test_util.hpp:40-48 random_field(dims, seed, mag): i.i.d. entries of
 * magnitude in [0.15, 1] * mag with random sign; host {3, n} */
mdg_status mdg_synth_random_field(mdg_dims3 d, uint64_t seed, float mag, float *out);
/* synth.cpp:92-192 make_synth_pair with SynthConfig defaults except seed and
 * max_disp: host outputs {n} images, {n} labels, {3, n} ground truth
 * (nullable).  Uses the device (scaling-and-squaring and warps). */
mdg_status mdg_synth_pair(mdg_dims3 d, uint64_t seed, float max_disp, float *fixed,
                          float *moving, int *labels_fixed, int *labels_moving, float *gt_field);

/* ====================== file formats (§8f rank 4) =========================
 * Host-side, no device needed.  Byte-identical to the reference's writers
 * and accepting what they write, with the same checks: raw volumes with a
 * JSON sidecar (io.hpp:23-34, io_raw.cpp) and the MDT2 checkpoint
 * (io.hpp:40-45, checkpoint.cpp).  Loaders called with a NULL data pointer
 * fill the header only (to size the buffer). */
#define MDG_RAW_F32 0
#define MDG_RAW_U16 1
typedef struct {
    mdg_dims3 dims;
    float spacing[3];
    int dtype;    /* MDG_RAW_F32 / MDG_RAW_U16 */
    int channels; /* 1 (volume, labels) or 3 (field) */
} mdg_raw_header;
/* load_raw_volume / load_raw_field / load_raw_labels (io_raw.cpp:142-169);
 * f32 payloads are checked finite; labels are u16 on disk, int here */
mdg_status mdg_raw_load_volume(const char *json_path, mdg_raw_header *hdr, float *out);
mdg_status mdg_raw_load_field(const char *json_path, mdg_raw_header *hdr, float *out);
mdg_status mdg_raw_load_labels(const char *json_path, mdg_raw_header *hdr, int *out);
/* load_nifti (io.hpp:36-38, nifti.cpp): single-file NIfTI-1 (u8 / i16 / f32,
 * scl_slope / scl_inter applied when slope != 0) into an f32 volume */
mdg_status mdg_nifti_load(const char *path, mdg_raw_header *hdr, float *out);
/* save_raw (io_raw.cpp:120-140): writes <base>.json and <base>.raw */
mdg_status mdg_raw_save_volume(const char *base, mdg_dims3 d, const float spacing[3],
                               const float *data);
mdg_status mdg_raw_save_field(const char *base, mdg_dims3 d, const float *data);
mdg_status mdg_raw_save_labels(const char *base, mdg_dims3 d, const float spacing[3],
                               const int *labels);

/* ModelConfig (engine.hpp:30-78) as stored in a checkpoint */
#define MDG_ENC_LEVELS 5
typedef struct {
    int base_channels;
    float leaky_slope;
    int heads_per_level[MDG_ENC_LEVELS]; /* coarse -> fine */
    int head_dim;
    int neighborhood;
    int diffeomorphic;
    int ss_steps;
} mdg_model_config;
mdg_status mdg_model_config_small_preset(mdg_model_config *cfg);
/* ModelParams::all_tensors layout for a config: tensor count, element counts
 * (sizes nullable); returns the total */
int64_t mdg_config_param_count(const mdg_model_config *cfg, int *ntensors, int64_t *sizes);
/* the reference's name of tensor i ("enc.l1.conv1.w", ..., "lvl4.reghead.b") */
mdg_status mdg_config_tensor_name(const mdg_model_config *cfg, int i, char *buf, int cap);
/* save_checkpoint / load_checkpoint (checkpoint.cpp:85-145): host tensors in
 * all_tensors order; load with tensors == NULL reads the config only */
mdg_status mdg_checkpoint_save(const char *path, const mdg_model_config *cfg,
                               const float *const *tensors);
mdg_status mdg_checkpoint_load(const char *path, mdg_model_config *cfg, float *const *tensors);

/* ---- the model object for any ModelConfig (engine.hpp:30-78, 268-311) ----
 * mdg_model_create / mdg_model_init above are this with the small preset and
 * Adam.  optimizer: OptimizerKind (engine.hpp:80) — MDG_OPT_ADAM (the
 * AdamOptimizer) or MDG_OPT_SGD (sgd_step); mdg_model_adam_step and
 * mdg_model_po_step apply the configured one.  Tensor sizes of a config:
 * mdg_config_param_count. */
#define MDG_OPT_ADAM 0
#define MDG_OPT_SGD 1
mdg_status mdg_model_init_cfg(const mdg_model_config *cfg, uint64_t seed,
                              float *const *params_host);
mdg_status mdg_model_create_cfg(const mdg_model_config *cfg, mdg_dims3 d, float *const *params,
                                float lambda, int ncc_window, int check_finite, int optimizer,
                                mdg_model **out);

/* pinned host memory for the host-buffer path */
void *mdg_host_alloc(size_t bytes);
void mdg_host_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* MDG_H */
