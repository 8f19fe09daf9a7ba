"""ctypes binding of ``include/mdg.h`` (libmdg.so, sm_100a).

The library is built in-tree (``paper_2403_16526_b200/libmdg.so``) by
``__graft_entry__.build()`` / ``make -C paper_2403_16526_b200/csrc``.  There is
no fallback: if the library is missing, importing the bindings raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmdg.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "mdg.h")

MDG_OK, MDG_EINVAL, MDG_ENUMERIC, MDG_ECUDA, MDG_EPARSE = 0, 1, 2, 3, 4
MDG_RAW_F32, MDG_RAW_U16 = 0, 1
ENC_LEVELS = 5
MDG_QK_POSMAJOR, MDG_QK_PLANAR = 0, 1


class Dims3(C.Structure):
    """{h, w, l} = extents along x, y, z (reference common.hpp:40-50)."""

    _fields_ = [("h", C.c_int), ("w", C.c_int), ("l", C.c_int)]

    def __iter__(self):
        return iter((self.h, self.w, self.l))

    def __repr__(self):
        return f"Dims3({self.h}, {self.w}, {self.l})"


MAX_LEVELS = 8


class PyramidConfig(C.Structure):
    """mdg_pyramid_config (ModelConfig + level geometry, engine.hpp:30-78)."""

    _fields_ = [("levels", C.c_int), ("heads", C.c_int * MAX_LEVELS),
                ("channels", C.c_int * MAX_LEVELS), ("dims", Dims3 * MAX_LEVELS),
                ("head_dim", C.c_int), ("neighborhood", C.c_int),
                ("diffeomorphic", C.c_int), ("ss_steps", C.c_int), ("check_finite", C.c_int)]


LEVEL_FIELDS = ("proj_w", "proj_b", "ln_g", "ln_b", "rel_bias", "rh_w", "rh_b")


class LevelParams(C.Structure):
    """mdg_level_params (LevelParams, engine.hpp:108-112)."""

    _fields_ = [(f, C.c_void_p) for f in LEVEL_FIELDS]


class LevelGrads(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in LEVEL_FIELDS]


BLOCK_FIELDS = ("w1", "b1", "g1", "be1", "w2", "b2", "g2", "be2")


class RawHeader(C.Structure):
    """mdg_raw_header."""

    _fields_ = [("dims", Dims3), ("spacing", C.c_float * 3), ("dtype", C.c_int),
                ("channels", C.c_int)]


class ModelConfigC(C.Structure):
    """mdg_model_config (ModelConfig engine.hpp:30-78 as stored in a checkpoint)."""

    _fields_ = [("base_channels", C.c_int), ("leaky_slope", C.c_float),
                ("heads_per_level", C.c_int * ENC_LEVELS), ("head_dim", C.c_int),
                ("neighborhood", C.c_int), ("diffeomorphic", C.c_int), ("ss_steps", C.c_int)]


class BlockParams(C.Structure):
    """mdg_block_params (ConvBlockParams, encoder.hpp:45-48)."""

    _fields_ = [(f, C.c_void_p) for f in BLOCK_FIELDS]


class BlockGrads(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in BLOCK_FIELDS]


_p = C.c_void_p  # device or host pointer
_i = C.c_int
_f = C.c_float
_st = C.c_int  # mdg_status

# name -> (restype, argtypes); mirrors include/mdg.h one to one
SIGNATURES = {
    "mdg_last_error": (C.c_char_p, []),
    "mdg_last_error_position": (None, [C.POINTER(_i)] * 4),
    "mdg_device_ok": (_i, []),
    "mdg_build_info": (C.c_char_p, []),
    "mdg_check_numeric": (_st, [Dims3, _p]),
    "mdg_launch_count": (C.c_int64, []),
    "mdg_window_offset": (_st, [_i, _i, C.POINTER(_i)]),
    "mdg_resolve_axis": (_st, [_p, _i, _i, _p, _p, _p, _p, _p]),
    "mdg_na_fused_fwd": (_st, [_p, _p, _p, Dims3, _i, _i, _i, _p, _p]),
    "mdg_na_fused_bwd": (_st, [_p, _p, _p, Dims3, _i, _i, _i, _p, _p, _p, _p, _p]),
    "mdg_subfields_fwd": (_st, [_p, Dims3, _i, _i, _p, _p]),
    "mdg_subfields_bwd": (_st, [Dims3, _i, _i, _p, _p, _p]),
    "mdg_subfields_check_rows": (_st, [_p, Dims3, _i, _i, _f, _p]),
    "mdg_warp_fwd": (_st, [_p, _i, Dims3, _p, _p, _p]),
    "mdg_warp_bwd": (_st, [_p, _i, Dims3, _p, _p, _p, _p, _p]),
    "mdg_upsample2_fwd": (_st, [_p, _i, Dims3, Dims3, _f, _p, _p]),
    "mdg_upsample2_bwd": (_st, [_i, Dims3, Dims3, _f, _p, _p, _p]),
    "mdg_conv3_fwd": (_st, [_p, _i, Dims3, _p, _p, _i, _p, _p]),
    "mdg_conv3_bwd": (_st, [_p, _i, Dims3, _p, _i, _p, _p, _p, _p, _p]),
    "mdg_warp_fwd_range": (_st, [_p, _i, Dims3, _p, _p, C.c_int64, C.c_int64, _p]),
    "mdg_warp_bwd_range": (_st, [_p, _i, Dims3, _p, _p, _p, _p, C.c_int64, C.c_int64, _p]),
    "mdg_warp_fwd_slab": (_st, [_p, _i, Dims3, _i, _i, _p, _p, _i, _i, _p]),
    "mdg_warp_bwd_slab": (_st, [_p, _i, Dims3, _i, _i, _p, _p, _p, _p, _i, _i, _p]),
    "mdg_ncc_slab_fwd": (_st, [_p, _p, Dims3, _i, _i, _i, _p, _p]),
    "mdg_ncc_slab_bwd": (_st, [_p, _p, Dims3, _i, _i, _i, C.c_float, _p, _p]),
    "mdg_ncc_slab_bwd_dev": (_st, [_p, _p, Dims3, _i, _i, _i, C.c_float, _p, _p, _p]),
    "mdg_warp_fwd_slab_async": (_st, [_p, _i, Dims3, _i, _i, _p, _p, _i, _i, _p, _p]),
    "mdg_warp_bwd_slab_async": (_st, [_p, _i, Dims3, _i, _i, _p, _p, _p, _p, _i, _i, _p, _p]),
    "mdg_in_slab_sums": (_st, [_p, _i, C.c_int64, _p, _p, _p]),
    "mdg_in_lrelu_apply": (_st, [_p, _i, C.c_int64, _p, _p, _p, _p, C.c_float, _p, _p]),
    "mdg_in_lrelu_bwd_sums": (_st, [_p, _p, _i, C.c_int64, _p, _p, _p, _p, C.c_float, _p, _p]),
    "mdg_in_lrelu_bwd_apply": (_st, [_p, _p, _i, C.c_int64, _p, _p, _p, _p, C.c_float, _p,
                                     C.c_int64, _p, _p]),
    "mdg_avgpool2_fwd": (_st, [_p, _i, Dims3, _p, _p]),
    "mdg_avgpool2_bwd": (_st, [_p, _i, Dims3, _p, _p]),
    "mdg_compose_fwd": (_st, [_p, _p, Dims3, _p, _p]),
    "mdg_compose_bwd": (_st, [_p, _p, Dims3, _p, _p, _p, _p]),
    "mdg_scaling_squaring_fwd": (_st, [_p, Dims3, _i, _p, _p, _p]),
    "mdg_scaling_squaring_bwd": (_st, [_p, Dims3, _i, _p, _p, _p]),
    "mdg_modet_fwd": (_st, [_p, _p, _p, Dims3, _i, _i, _i, _i, _p, _p, _p, _p]),
    "mdg_modet_bwd": (_st, [_p, _p, _p, _p, _p, _p, Dims3, _i, _i, _i, _i, _p, _p, _p, _i, _p]),
    "mdg_project_qk_fwd": (_st, [_p, _p, _i, C.c_int64, _p, _p, _p, _p, _i, _i, _p, _p, _p]),
    "mdg_project_qk_bwd": (_st, [_p, _p, _i, C.c_int64, _p, _p, _p, _i, _i, _p, _p, _p, _p,
                                 _p, _p, _p, _p, _p]),
    "mdg_total_loss_fwd": (_st, [_p, _p, _p, Dims3, _i, _f, _p, _p, _p]),
    "mdg_total_loss_bwd": (_st, [_p, _p, _p, Dims3, _i, _f, _f, _p, _p, _p]),
    "mdg_adam_step": (_st, [_p, _p, _p, _p, C.c_int64, C.c_double, C.c_double, C.c_double,
                            C.c_double, C.c_int64, _p]),
    "mdg_sgd_step": (_st, [_p, _p, C.c_int64, C.c_double, _p]),
    "mdg_warp_labels": (_st, [_p, Dims3, _p, _p, _p]),
    "mdg_mean_dice": (_st, [_p, _p, C.c_int64, _i, C.POINTER(C.c_double), _p]),
    "mdg_encoder_conv3_fwd": (_st, [_p, _i, Dims3, _p, _p, _i, _p, _p]),
    "mdg_encoder_conv3_bwd": (_st, [_p, _i, Dims3, _p, _i, _p, _p, _p, _p, _p]),
    "mdg_encoder_create": (_st, [Dims3, _i, _i, _f, C.POINTER(_p)]),
    "mdg_encoder_destroy": (None, [_p]),
    "mdg_encoder_forward": (_st, [_p, _p, C.POINTER(BlockParams), C.POINTER(_p), _p]),
    "mdg_encoder_backward": (_st, [_p, C.POINTER(_p), C.POINTER(BlockGrads), _p, _p]),
    "mdg_model_param_count": (C.c_int64, [C.POINTER(_i), C.POINTER(C.c_int64)]),
    "mdg_model_init": (_st, [C.c_uint64, C.POINTER(_p)]),
    "mdg_model_create": (_st, [Dims3, C.POINTER(_p), _f, _i, _i, C.POINTER(_p)]),
    "mdg_model_destroy": (None, [_p]),
    "mdg_model_init_cfg": (_st, [C.POINTER(ModelConfigC), C.c_uint64, C.POINTER(_p)]),
    "mdg_model_create_cfg": (_st, [C.POINTER(ModelConfigC), Dims3, C.POINTER(_p), _f, _i, _i, _i,
                                   C.POINTER(_p)]),
    "mdg_model_grads": (C.POINTER(_p), [_p]),
    "mdg_model_loss_step": (_st, [_p, _p, _p, _i, _p, _p, _p]),
    "mdg_model_adam_step": (_st, [_p, C.c_double, _p]),
    "mdg_model_po_step": (_st, [_p, _p, _p, C.c_double, _p, _p]),
    "mdg_model_phi": (_p, [_p]),
    "mdg_pyramid_create": (_st, [C.POINTER(PyramidConfig), C.POINTER(_p)]),
    "mdg_pyramid_destroy": (None, [_p]),
    "mdg_pyramid_forward": (_st, [_p, C.POINTER(_p), C.POINTER(_p), C.POINTER(LevelParams), _p,
                                  C.POINTER(_p), _p]),
    "mdg_pyramid_backward": (_st, [_p, _p, C.POINTER(LevelGrads), C.POINTER(_p), C.POINTER(_p),
                                   _p]),
    "mdg_pyramid_bytes": (C.c_int64, [_p]),
    "mdg_qk_posmajor_to_planar": (_st, [_p, C.c_int64, _i, _p, _p]),
    "mdg_qk_planar_to_posmajor": (_st, [_p, C.c_int64, _i, _p, _p]),
    "mdg_na_fused_fwd_host": (_st, [_p, _p, _p, Dims3, _i, _i, _i, _p]),
    "mdg_na_fused_bwd_host": (_st, [_p, _p, _p, Dims3, _i, _i, _i, _p, _p, _p, _p]),
    "mdg_subfields_fwd_host": (_st, [_p, Dims3, _i, _i, _p]),
    "mdg_subfields_bwd_host": (_st, [Dims3, _i, _i, _p, _p]),
    "mdg_upsample2_fwd_host": (_st, [_p, _i, Dims3, Dims3, _f, _p]),
    "mdg_upsample2_bwd_host": (_st, [_i, Dims3, Dims3, _f, _p, _p]),
    "mdg_conv3_fwd_host": (_st, [_p, _i, Dims3, _p, _p, _i, _p]),
    "mdg_conv3_bwd_host": (_st, [_p, _i, Dims3, _p, _i, _p, _p, _p, _p]),
    "mdg_modet_fwd_host": (_st, [_p, _p, _p, Dims3, _i, _i, _i, _i, _p, _p]),
    "mdg_modet_bwd_host": (_st, [_p, _p, _p, _p, _p, _p, Dims3, _i, _i, _i, _i, _p, _p, _p, _i]),
    "mdg_warp_fwd_host": (_st, [_p, _i, Dims3, _p, _p]),
    "mdg_warp_bwd_host": (_st, [_p, _i, Dims3, _p, _p, _p, _p]),
    "mdg_raw_load_volume": (_st, [C.c_char_p, C.POINTER(RawHeader), _p]),
    "mdg_raw_load_field": (_st, [C.c_char_p, C.POINTER(RawHeader), _p]),
    "mdg_raw_load_labels": (_st, [C.c_char_p, C.POINTER(RawHeader), _p]),
    "mdg_nifti_load": (_st, [C.c_char_p, C.POINTER(RawHeader), _p]),
    "mdg_raw_save_volume": (_st, [C.c_char_p, Dims3, C.POINTER(C.c_float), _p]),
    "mdg_raw_save_field": (_st, [C.c_char_p, Dims3, _p]),
    "mdg_raw_save_labels": (_st, [C.c_char_p, Dims3, C.POINTER(C.c_float), _p]),
    "mdg_model_config_small_preset": (_st, [C.POINTER(ModelConfigC)]),
    "mdg_config_param_count": (C.c_int64, [C.POINTER(ModelConfigC), C.POINTER(_i),
                                           C.POINTER(C.c_int64)]),
    "mdg_config_tensor_name": (_st, [C.POINTER(ModelConfigC), _i, C.c_char_p, _i]),
    "mdg_checkpoint_save": (_st, [C.c_char_p, C.POINTER(ModelConfigC), C.POINTER(_p)]),
    "mdg_checkpoint_load": (_st, [C.c_char_p, C.POINTER(ModelConfigC), C.POINTER(_p)]),
    "mdg_rng_new": (_p, [C.c_uint64]),
    "mdg_rng_free": (None, [_p]),
    "mdg_rng_fill_uniform": (None, [_p, _p, C.c_int64, C.c_double, C.c_double]),
    "mdg_rng_fill_normal": (None, [_p, _p, C.c_int64, C.c_double, C.c_double]),
    "mdg_synth_smooth_velocity": (_st, [Dims3, C.c_uint64, _f, _f, _p]),
    "mdg_synth_random_field": (_st, [Dims3, C.c_uint64, _f, _p]),
    "mdg_synth_pair": (_st, [Dims3, C.c_uint64, _f, _p, _p, _p, _p, _p]),
    "mdg_set_deterministic": (_i, [_i]),
    "mdg_get_deterministic": (_i, []),
    "mdg_host_alloc": (_p, [C.c_size_t]),
    "mdg_host_free": (None, [_p]),
}


class _Lib:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise ImportError(
                f"libmdg.so not found at {path}: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)


_LIB = None


def lib() -> _Lib:
    global _LIB
    if _LIB is None:
        _LIB = _Lib()
    return _LIB


def header_symbols(path: str = HEADER):
    """Function names declared in include/mdg.h (for the export test)."""
    import re

    txt = open(path).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mdg_[a-z0-9_]+)\s*\(", txt)))
