"""CPU: the C-ABI library loads, exports every symbol include/mdg.h declares,
and its host-side logic (argument validation, error mapping, exact index
helpers, the synthetic-input RNG) behaves like the reference — no GPU needed
(validation returns before any CUDA call)."""
import ctypes as C
import subprocess

import numpy as np
import pytest

import pyoracle
from paper_2403_16526_b200 import _capi, ops


def test_library_exports_every_header_symbol():
    syms = _capi.header_symbols()
    assert len(syms) >= 35
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # and the ctypes table binds exactly the header
    assert sorted(_capi.SIGNATURES) == syms


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90", "sm_103"):
        assert other + "." not in out


def test_window_offset_matches_reference_order(oracle):
    for nb in (3, 5, 7):
        for o in range(nb ** 3):
            assert ops.window_offset(o, nb) == oracle.window_offset(o, nb)
    with pytest.raises(ops.InvalidInput):
        ops.window_offset(0, 4)


def test_validation_errors_map_to_invalid_input():
    L = _capi.lib()
    d = _capi.Dims3(4, 4, 4)
    # attention.hpp:48-53
    assert L.mdg_modet_fwd(None, None, None, d, 1, 6, 4, 0, None, None, None, None) == 1
    assert "odd" in L.mdg_last_error().decode()
    assert L.mdg_na_fused_fwd(None, None, None, d, 0, 6, 3, None, None) == 1
    assert "positive" in L.mdg_last_error().decode()
    # sampling.hpp:266-271
    assert L.mdg_upsample2_fwd(None, 3, d, _capi.Dims3(12, 8, 8), 2.0, None, None) == 1
    assert "doubling range" in L.mdg_last_error().decode()
    assert L.mdg_scaling_squaring_fwd(None, d, 0, None, None, None) == 1
    assert "steps" in L.mdg_last_error().decode()
    assert L.mdg_conv3_fwd(None, 0, d, None, None, 3, None, None) == 1
    # empty volumes are a no-op, like the reference's empty loops
    assert L.mdg_warp_fwd(None, 2, _capi.Dims3(0, 4, 4), None, None, None) == 0


def test_python_face_refuses_cpu_tensors():
    import torch

    x = torch.zeros(8, 6)
    with pytest.raises(ops.InvalidInput, match="CUDA"):
        ops.kern.na_fused_fwd(x, x, torch.zeros(1, 27), (2, 2, 2), 1, 6, 3, torch.zeros(1, 8, 27))


def test_rng_stream_bit_identical_to_reference_rng():
    r1 = ops.Rng(5)
    a = r1.uniform(1001, -1.0, 1.0).numpy()
    b = r1.normal(777).numpy()
    c = r1.uniform(3, -0.5, 0.5).numpy()
    r2 = pyoracle.Rng(5)
    assert np.array_equal(a, r2.uniform(1001, -1.0, 1.0).astype(np.float32))
    assert np.array_equal(b, r2.normal(777).astype(np.float32))
    assert np.array_equal(c, r2.uniform(3, -0.5, 0.5).astype(np.float32))


def test_host_alloc_roundtrip_api_present():
    L = _capi.lib()
    assert isinstance(L.mdg_build_info().decode(), str)
    assert L.mdg_launch_count() >= 0


def test_slab_entry_points_validate_before_touching_the_device():
    """The depth-slab entry points (slab warps, slab NCC, slab instance norm)
    refuse inconsistent geometry with MDG_EINVAL and a message, no GPU."""
    L = _capi.lib()
    d = _capi.Dims3(8, 8, 32)
    # the input window must cover the slab's planes
    assert L.mdg_warp_fwd_slab(None, 2, d, 6, 20, None, None, 4, 12, None) == 1
    assert "cover" in L.mdg_last_error().decode()
    assert L.mdg_warp_bwd_slab(None, 2, d, 0, 40, None, None, None, None, 4, 12, None) == 1
    assert L.mdg_warp_fwd_slab(None, 2, d, 0, 32, None, None, 12, 4, None) == 1
    assert "plane range" in L.mdg_last_error().decode()
    assert L.mdg_warp_fwd_slab_async(None, 2, d, 0, 32, None, None, 0, 32, None, None) == 1
    assert "error word" in L.mdg_last_error().decode()
    # an empty slab is a no-op
    assert L.mdg_warp_fwd_slab(None, 2, d, 0, 32, None, None, 5, 5, None) == 0
    # slab NCC: odd window, own planes inside the halos, in-volume range
    e = _capi.Dims3(8, 8, 24)
    assert L.mdg_ncc_slab_fwd(None, None, e, 8, 4, 20, None, None) == 1
    assert "odd" in L.mdg_last_error().decode()
    assert L.mdg_ncc_slab_fwd(None, None, _capi.Dims3(8, 8, 8), 9, 0, 8, None, None) == 1
    assert "own planes" in L.mdg_last_error().decode()
    assert L.mdg_ncc_slab_fwd(None, None, e, 9, 6, 24, None, None) == 1
    assert "in-volume" in L.mdg_last_error().decode()
    assert L.mdg_ncc_slab_bwd_dev(None, None, e, 9, 4, 20, 1.0, None, None, None) == 1
    # slab instance norm
    assert L.mdg_in_slab_sums(None, 0, 16, None, None, None) == 1
    assert "invalid sizes" in L.mdg_last_error().decode()
    assert L.mdg_in_lrelu_bwd_apply(None, None, 2, 16, None, None, None, None, 0.2, None, 8,
                                    None, None) == 1
