// mdreg_b200.hpp — binds the UNMODIFIED mdreg reference to libmdg (B200).
//
// Force-include it into every translation unit of a reference build
//     g++ -std=c++20 -DMDREG_B200 -include integration/mdreg_b200.hpp \
//         -I<mdreg>/include -Iinclude ... -Lpaper_2403_16526_b200 -lmdg
// and the reference's own operators (op_na_fused, op_subfields, op_warp,
// op_upsample_field_2x, op_conv3 / op_reghead_fuse, plain warp / compose,
// hence build_pipeline, run_loss_step and pairwise_optimize) run their float
// kernels on the GPU.  Nothing in the reference tree is edited: the header
// pulls in the reference's primary kern:: templates and declares explicit
// specialisations for T = float before any other header instantiates them.
//
//   kern::na_fused_fwd<float>   attention.hpp:83   -> mdg_na_fused_fwd_host
//   kern::na_fused_bwd<float>   attention.hpp:127  -> mdg_na_fused_bwd_host
//   kern::subfields_fwd<float>  attention.hpp:282  -> mdg_subfields_fwd_host
//   kern::subfields_bwd<float>  attention.hpp:301  -> mdg_subfields_bwd_host
//   kern::warp_fwd<float>       sampling.hpp:123   -> mdg_warp_fwd_host
//   kern::warp_bwd<float>       sampling.hpp:139   -> mdg_warp_bwd_host
//   op_upsample_field_2x<float> ops.hpp:258        -> mdg_upsample2_fwd_host (*)
//   kern::upsample2_bwd<float>  sampling.hpp:245   -> mdg_upsample2_bwd_host
// (*) kern::upsample2_fwd<float> itself cannot be specialised from outside:
//     sampling.hpp's own inline upsample_field_2x (:303-308, the generators'
//     helper) instantiates it inside the header.  The tape operator that
//     build_pipeline uses is specialised instead (same body, GPU forward).
//   kern::conv3_fwd<float>      ops.hpp:58         -> mdg_conv3_fwd_host
//   kern::conv3_bwd<float>      ops.hpp:77         -> mdg_conv3_bwd_host
//
// Semantics are the reference's: outputs overwritten, gradients accumulated,
// NULL gradients skipped; MDG_EINVAL / MDG_ENUMERIC / MDG_EPARSE come back as
// the reference's invalid_input / numeric_error / parse_error (same messages,
// common.hpp:25-38).  The calls are synchronous and host-buffer based, exactly
// like the CPU functions they replace; the device-resident pipeline
// (mdg_pyramid_*, mdg_model_*) is the fast path for whole iterations.
#pragma once

#ifndef MDREG_B200
#error "mdreg_b200.hpp binds the reference to libmdg: compile with -DMDREG_B200"
#endif

#include <stdexcept>

#include "mdg.h"
#include "mdreg/attention.hpp"  // + ops.hpp, sampling.hpp, tape.hpp: the primary templates

namespace mdreg {
namespace b200 {
// the reference guarantees bitwise-repeatable runs (test_engine.cpp:194-213):
// the binding switches libmdg to its deterministic mode at load time
inline const bool deterministic_on = (mdg_set_deterministic(1), true);

inline void check(mdg_status s) {
    switch (s) {
        case MDG_OK: return;
        case MDG_EINVAL: throw invalid_input(mdg_last_error());
        case MDG_ENUMERIC: throw numeric_error(mdg_last_error());
        case MDG_EPARSE: throw parse_error(mdg_last_error());
        default: throw std::runtime_error(mdg_last_error());
    }
}
inline mdg_dims3 dims(const Dims3 &d) { return mdg_dims3{d.h, d.w, d.l}; }
}  // namespace b200

namespace kern {
template <>
inline void na_fused_fwd<float>(const float *Q, const float *K, const float *B, const Dims3 &d,
                                int S, int hd, int nb, float *out, MemCounter *) {
    b200::check(mdg_na_fused_fwd_host(Q, K, B, b200::dims(d), S, hd, nb, out));
}
template <>
inline void na_fused_bwd<float>(const float *Q, const float *K, const float *W, const Dims3 &d,
                                int S, int hd, int nb, const float *gW, float *gQ, float *gK,
                                float *gB) {
    b200::check(mdg_na_fused_bwd_host(Q, K, W, b200::dims(d), S, hd, nb, gW, gQ, gK, gB));
}
template <>
inline void subfields_fwd<float>(const float *W, const Dims3 &d, int S, int nb, float *out) {
    b200::check(mdg_subfields_fwd_host(W, b200::dims(d), S, nb, out));
}
template <>
inline void subfields_bwd<float>(const Dims3 &d, int S, int nb, const float *gout, float *gW) {
    b200::check(mdg_subfields_bwd_host(b200::dims(d), S, nb, gout, gW));
}
template <>
inline void warp_fwd<float>(const float *in, int channels, const Dims3 &d, const float *field,
                            float *out) {
    b200::check(mdg_warp_fwd_host(in, channels, b200::dims(d), field, out));
}
template <>
inline void warp_bwd<float>(const float *in, int channels, const Dims3 &d, const float *field,
                            const float *gout, float *gin, float *gfield) {
    b200::check(mdg_warp_bwd_host(in, channels, b200::dims(d), field, gout, gin, gfield));
}
template <>
inline void upsample2_bwd<float>(int channels, const Dims3 &d, const Dims3 &td, float scale,
                                 const float *gout, float *gin) {
    b200::check(mdg_upsample2_bwd_host(channels, b200::dims(d), b200::dims(td), scale, gout, gin));
}
template <>
inline void conv3_fwd<float>(const float *in, int ic, const Dims3 &d, const float *k,
                             const float *bias, int oc, float *out) {
    b200::check(mdg_conv3_fwd_host(in, ic, b200::dims(d), k, bias, oc, out));
}
template <>
inline void conv3_bwd<float>(const float *in, int ic, const Dims3 &d, const float *k, int oc,
                             const float *gout, float *gin, float *gk, float *gbias) {
    b200::check(mdg_conv3_bwd_host(in, ic, b200::dims(d), k, oc, gout, gin, gk, gbias));
}
}  // namespace kern

// ops.hpp:256-271 with the forward on the GPU (the backward node calls the
// specialised kern::upsample2_bwd<float>)
template <>
inline Var op_upsample_field_2x<float>(Tape<float> &t, Var field, Dims3 target) {
    const Tensor<float> &vf = t.value(field);
    const Dims3 d = spatial_dims(vf.shape);
    check_upsample_target(d, target);
    const int c = vf.shape[0];
    Tensor<float> out({c, target.h, target.w, target.l});
    b200::check(mdg_upsample2_fwd_host(vf.data.data(), c, b200::dims(d), b200::dims(target),
                                       2.0f, out.data.data()));
    Var o = t.push(std::move(out), "upsample_field_2x");
    t.set_backward(o, [o, field, c, d, target](Tape<float> &tt) {
        kern::upsample2_bwd(c, d, target, 2.0f, tt.grad(o).data.data(),
                            tt.grad(field).data.data());
    });
    return o;
}
}  // namespace mdreg
