"""GPU parity of warp / compose / upsample / RegHead conv3 / scaling-squaring.

Forward results and every gather-form gradient are BIT-IDENTICAL to the CPU
reference (same fp32 evaluation order, no FMA contraction); the image-side
scatter gradients (warp gin, compose gprev) are fp32 atomic scatters by
default, checked to |d| <= 1e-5 + 1e-4|ref|; in deterministic mode they are a
64-bit fixed-point scatter (whole volume) or gathered per target
(warp_gather.cu, voxel ranges), bit-identical from run to run (the gather
also bit-identical to the reference on the exact path crowded cells take).  The integer corner logic (resolve_axis) is checked
bit-for-bit on the device.
"""
import numpy as np
import pytest
import torch

import pyoracle
from _util import f32, load_golden, random_feature_map, random_field, rel_close
from paper_2403_16526_b200 import ops

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def test_resolve_axis_bit_exact_on_device(cuda, oracle):
    r = pyoracle.Rng(3)
    xs = np.concatenate([
        f32(r.uniform(20000, -3.0, 12.0)),
        np.array([-1.0, -0.0, 0.0, 1e-8, 0.5, 1.0, 4.0, 4.5, 5.0, 5.0000005, 9.0, 8.999999,
                  2 ** -126, -(2 ** -126), 1e30, -1e30], np.float32),
        np.arange(0, 10, 0.5, dtype=np.float32)])
    xs = f32(xs)
    for dim in (1, 2, 3, 5, 10):
        i0, i1, f, live = (host(t) for t in ops.kern.resolve_axis(dev(xs), dim))
        ref = np.array([oracle.resolve_axis(float(x), dim) for x in xs], dtype=object)
        assert np.array_equal(i0, ref[:, 0].astype(np.int32)), dim
        assert np.array_equal(i1, ref[:, 1].astype(np.int32)), dim
        assert np.array_equal(f, ref[:, 2].astype(np.float32)), dim
        assert np.array_equal(live, ref[:, 3].astype(np.int32)), dim


@pytest.mark.parametrize("name", ["warp_7x6x5_c3_m1p5", "warp_6x5x4_c2_m6", "warp_5x1x4_c1_m1"])
def test_warp_matches_golden(cuda, name):
    g = load_golden(name)
    vol, fld = dev(g["vol"]), dev(g["field"])
    assert np.array_equal(host(ops.warp(vol, fld)), g["out"])
    gin, gfield = ops.warp_bwd(vol, fld, dev(g["gout"]))
    assert np.array_equal(host(gfield), g["gfield"])
    assert rel_close(host(gin), g["gin"])


def test_warp_randomised_bit_exact(cuda, oracle):
    seeds = pyoracle.Rng(11)
    for trial in range(16):
        dims = tuple(int(seeds.uniform_int(1, 12)) for _ in range(3))
        C = seeds.uniform_int(1, 9)
        mag = [0.3, 1.5, 4.0, 20.0][trial % 4]
        vol = random_feature_map(C, dims, 100 + trial)
        fld = random_field(dims, 200 + trial, mag)
        gout = random_feature_map(C, dims, 300 + trial)
        gout[:, ::2] = 0.0  # exercise the g == 0 skip (sampling.hpp:152)
        out = host(ops.warp(dev(vol), dev(fld)))
        assert np.array_equal(out, oracle.warp_fwd(vol, fld)), (trial, dims, C)
        gin, gfield = ops.warp_bwd(dev(vol), dev(fld), dev(gout))
        rgin, rgfield = oracle.warp_bwd(vol, fld, gout)
        assert np.array_equal(host(gfield), rgfield), (trial, dims)
        assert rel_close(host(gin), rgin), (trial, dims)


def test_warp_zero_field_identity_and_accumulate(cuda):
    v = dev(random_feature_map(3, (5, 6, 4), 3))
    z = torch.zeros(3, 4, 6, 5, device="cuda")
    assert torch.equal(ops.warp(v, z), v)
    # backward accumulates into existing gradients (sampling.hpp:153-164)
    g = dev(random_feature_map(3, (5, 6, 4), 4))
    gin0 = torch.ones_like(v)
    gin, _ = ops.warp_bwd(v, z, g, gin=gin0.clone(), want_gfield=False)
    assert torch.allclose(gin, gin0 + g, atol=1e-6)


def test_compose_matches_golden(cuda):
    g = load_golden("compose_7x6x5")
    prev, res = dev(g["prev"]), dev(g["res"])
    assert np.array_equal(host(ops.compose(prev, res)), g["out"])
    gp, gr = ops.compose_bwd(prev, res, dev(g["gout"]))
    assert np.array_equal(host(gr), g["gres"])
    assert rel_close(host(gp), g["gprev"])


@pytest.mark.parametrize("name", ["up_4x3x3_to_8x6x5", "up_4x4x4_to_7x8x9", "up_1x2x2_to_2x3x4"])
def test_upsample_matches_golden(cuda, name):
    g = load_golden(name)
    d, td = tuple(int(v) for v in g["dims"]), tuple(int(v) for v in g["tdims"])
    y = ops.upsample_field_2x(dev(g["x"]), td)
    assert np.array_equal(host(y), g["y"])
    gin = ops.upsample_field_2x_bwd(dev(g["gout"]), d, td)
    assert rel_close(host(gin), g["gin"], 1e-6, 1e-5)


def test_upsample_rejects_bad_target(cuda):
    f = torch.zeros(3, 4, 4, 4, device="cuda")
    with pytest.raises(ops.InvalidInput, match="doubling range"):
        ops.upsample_field_2x(f, (12, 8, 8))
    ops.upsample_field_2x(f, (7, 8, 9))


def test_upsample_randomised(cuda, oracle):
    seeds = pyoracle.Rng(5)
    for trial in range(10):
        d = tuple(int(seeds.uniform_int(1, 9)) for _ in range(3))
        td = tuple(2 * v + seeds.uniform_int(-1, 1) if v > 1 else 2 * v for v in d)
        x = random_feature_map(3, d, 10 + trial)
        g = random_feature_map(3, td, 20 + trial)
        assert np.array_equal(host(ops.upsample_field_2x(dev(x), td)),
                              oracle.upsample2_fwd(x, td))
        assert rel_close(host(ops.upsample_field_2x_bwd(dev(g), d, td)),
                         oracle.upsample2_bwd(g, d), 1e-6, 1e-5)


def test_conv3_matches_golden(cuda):
    g = load_golden("conv3_6x5x4_ic6_oc3")
    x, k, b = dev(g["x"]), dev(g["k"]), dev(g["b"])
    assert np.array_equal(host(ops.conv3(x, k, b)), g["y"])
    gin, gk, gb = ops.conv3_bwd(x, k, dev(g["gout"]))
    assert np.array_equal(host(gin), g["gin"])
    assert rel_close(host(gk), g["gk"], 1e-5, 1e-4)
    assert rel_close(host(gb), g["gb"], 1e-5, 1e-4)


def test_conv3_reghead_shapes_randomised(cuda, oracle):
    for S, d in ((1, (9, 8, 7)), (2, (6, 7, 5)), (8, (4, 3, 5)), (4, (1, 1, 1)), (2, (40, 11, 3)),
                 (3, (33, 17, 2))):
        x = random_feature_map(3 * S, d, 7 * S)
        k = f32(pyoracle.Rng(S).normal(3 * 3 * S * 27, 0, 0.2).reshape(3, 3 * S, 3, 3, 3))
        b = f32(pyoracle.Rng(S + 1).normal(3))
        g = random_feature_map(3, d, 9 * S)
        assert np.array_equal(host(ops.conv3(dev(x), dev(k), dev(b))), oracle.conv3_fwd(x, k, b))
        gin, gk, gb = ops.conv3_bwd(dev(x), dev(k), dev(g))
        rgin, rgk, rgb = oracle.conv3_bwd(x, k, g)
        assert np.array_equal(host(gin), rgin)
        assert rel_close(host(gk), rgk, 1e-5, 1e-4) and rel_close(host(gb), rgb, 1e-5, 1e-4)


def test_scaling_squaring_golden_and_backward(cuda, oracle):
    g = load_golden("ss_8x7x6_t7")
    v = dev(g["vel"])
    out, saved = ops.scaling_squaring(v, 7, keep=True)
    assert np.array_equal(host(out), g["out"])
    # backward = chain of compose backwards (tape semantics, reghead.hpp:52-57)
    gout = random_feature_map(3, (8, 7, 6), 5)
    gv = host(ops.scaling_squaring_bwd(saved, 7, dev(gout)))
    sv = host(saved)
    G = gout.copy()
    for i in range(6, -1, -1):
        gp, gr = oracle.compose_bwd(f32(sv[i]), f32(sv[i]), f32(G))
        G = f32(gp + gr)
    assert rel_close(gv, G / 128.0, 1e-5, 1e-4)


@pytest.mark.slow
def test_north_star_size_warp_c8(cuda, oracle):
    """Warp fwd+bwd at 160x192x224 with C=8 features and the reference's smooth
    benchmark field (make_smooth_velocity seed 11, 2 vox, sigma 4) is
    generated here from the random stream; fwd and gfield bit-exact, gin within
    tolerance."""
    dims = (160, 192, 224)
    vol = random_feature_map(8, dims, 21)
    fld = random_field(dims, 22, 2.0)
    gout = random_feature_map(8, dims, 23)
    vd, fd, gd = dev(vol), dev(fld), dev(gout)
    out = host(ops.warp(vd, fd))
    gin, gfield = ops.warp_bwd(vd, fd, gd)
    assert np.array_equal(out, oracle.warp_fwd(vol, fld))
    rgin, rgfield = oracle.warp_bwd(vol, fld, gout)
    assert np.array_equal(host(gfield), rgfield)
    assert rel_close(host(gin), rgin)


@pytest.mark.parametrize("reach", ["small", "far", "nonfinite"])
@pytest.mark.parametrize("C", [8, 3, 5])
def test_pipelined_warp_host_calls_match_device(cuda, C, reach):
    """>= 1M voxels: warp_fwd_host / warp_bwd_host run the reach-aware z-chunk
    pipeline (field first, per-chunk sampled z range on the device, input
    chunks streamed, the scattered gradient downloaded as rows become final,
    contributions added into the caller's host accumulators by host threads).
    out and gfield are bit-identical to the device call; gin (fp32 atomics) to
    scatter tolerance.  `reach`: small field, far-reaching z displacements
    (several chunks, both directions), and non-finite entries."""
    import ctypes as C_

    from paper_2403_16526_b200 import _capi

    dims = (128, 96, 100)
    h, w, l = dims
    r = np.random.default_rng(C)
    vol = f32(r.standard_normal((C, l, w, h)))
    fld = f32(r.uniform(-2.5, 2.5, (3, l, w, h)))
    if reach == "far":
        fld[2, 10:20] += 37.0    # forward several chunks
        fld[2, 70:75] -= 55.5    # backward several chunks
        fld[2, 95:] += 1e9       # far outside (clamped)
    elif reach == "nonfinite":
        fld[2, 40, 3, 5] = np.nan
        fld[0, 60, 7, 9] = np.inf
    g = f32(r.standard_normal((C, l, w, h)))
    gin0 = f32(r.standard_normal((C, l, w, h)))
    gf0 = f32(r.standard_normal((3, l, w, h)))
    out_d = host(ops.warp(dev(vol), dev(fld)))
    gin_d, gf_d = ops.warp_bwd(dev(vol), dev(fld), dev(g), gin=dev(gin0), gfield=dev(gf0))
    gin_d, gf_d = host(gin_d), host(gf_d)
    L = _capi.lib()
    p = lambda a: a.ctypes.data_as(C_.c_void_p)  # noqa: E731
    d3 = _capi.Dims3(*dims)
    out = np.zeros_like(vol)
    assert L.mdg_warp_fwd_host(p(vol), C, d3, p(fld), p(out)) == 0
    assert np.array_equal(out, out_d, equal_nan=True)
    gin, gf = gin0.copy(), gf0.copy()
    assert L.mdg_warp_bwd_host(p(vol), C, d3, p(fld), p(g), p(gin), p(gf)) == 0
    assert np.array_equal(gf, gf_d, equal_nan=True)
    np.testing.assert_allclose(gin, gin_d, rtol=1e-4, atol=1e-5, equal_nan=True)


# ------------------------------------------------ deterministic gin gather
# (deterministic mode, mdg_set_deterministic: gathered per target; the default
# mode scatters with float atomics and is covered by the tests above)
def _gin_twice(vol, fld, gout):
    a, _ = ops.warp_bwd(vol, fld, gout)
    b, _ = ops.warp_bwd(vol, fld, gout)
    return host(a), host(b)


@pytest.mark.parametrize("kind", ["smooth", "random", "contracting", "far"])
def test_warp_gin_gather_deterministic_and_correct(cuda, oracle, ref, deterministic, kind):
    """gin from the per-target gather: identical from run to run (bitwise),
    within tolerance of the reference scatter, for a smooth field, the i.i.d.
    random field (|phi| <= 2), a contracting field (x -> x/3: crowded cells
    take the exact reference-order path) and a far field (|phi| = 9 > the
    gather's reach of 4: the atomic scatter fallback, correct but not
    repeatable)."""
    dims = (37, 21, 19)
    h, w, l = dims
    C = 3
    vol = random_feature_map(C, dims, 5)
    if kind == "smooth":
        fld = ref.make_smooth_velocity(dims, 11, 2.0, 3.0)
    elif kind == "random":
        fld = random_field(dims, 12, 2.0)
    elif kind == "contracting":
        zz, yy, xx = np.meshgrid(np.arange(l), np.arange(w), np.arange(h), indexing="ij")
        # x, y -> a third of their distance from the centre: ~9 sources per
        # cell in the middle (> the 4-entry lists: exact path)
        fld = f32(np.stack([-(2.0 / 3.0) * (xx - h / 2), -(2.0 / 3.0) * (yy - w / 2),
                            0.25 * np.ones_like(zz, dtype=np.float64)]))
        fld = f32(np.clip(fld, -3.9, 3.9))  # within the gather's reach (4)
    else:
        fld = f32(np.full((3, l, w, h), 9.0))
        fld[0] *= -1.0
    gout = random_feature_map(C, dims, 6)
    gout[:, 3, 4, :5] = 0.0  # g == 0 channels are skipped like the reference does
    want, _ = oracle.warp_bwd(vol, fld, gout)
    a, b = _gin_twice(dev(vol), dev(fld), dev(gout))
    assert rel_close(a, want), np.abs(a - want).max()
    if kind != "far":
        assert np.array_equal(a, b)


@pytest.mark.parametrize("C", [1, 3, 5, 8, 16])
@pytest.mark.parametrize("kind", ["smooth", "far"])
def test_warp_gin_fixed_point_whole_volume(cuda, oracle, deterministic, C, kind):
    """Deterministic mode, whole volume: gin by the 64-bit fixed-point scatter
    (integer REDs, order independent): within tolerance of the reference and
    bit-identical from run to run, also for a field beyond the range
    gather's reach (|phi| = 9) and for channel counts without an unrolled
    kernel (5: the runtime loop)."""
    dims = (37, 21, 19)
    h, w, l = dims
    vol = random_feature_map(C, dims, 15)
    if kind == "smooth":
        fld = random_field(dims, 16, 1.5)
    else:
        fld = f32(np.full((3, l, w, h), 9.0))
        fld[1] *= -1.0
    gout = random_feature_map(C, dims, 17)
    want, want_gf = oracle.warp_bwd(vol, fld, gout)
    a, b = _gin_twice(dev(vol), dev(fld), dev(gout))
    assert rel_close(a, want), np.abs(a - want).max()
    assert np.array_equal(a, b)
    _, gf = ops.warp_bwd(dev(vol), dev(fld), dev(gout))
    assert np.array_equal(host(gf), want_gf)  # gfield stays bit-exact


@pytest.mark.parametrize("scale", [1e30, 1e-30, 1e-41])
def test_warp_gin_fixed_point_extreme_magnitudes(cuda, oracle, deterministic, scale):
    """The fixed-point scale follows each channel's max |gout| over any float
    exponent (huge, tiny, subnormal gradients): relative parity with the
    reference scatter and run-to-run identity."""
    dims = (20, 12, 10)
    vol = random_feature_map(3, dims, 24)
    fld = random_field(dims, 25, 1.5)
    gout = f32(random_feature_map(3, dims, 26) * np.float32(scale))
    gout[1] *= np.float32(1e-3)  # channels of different magnitude
    want, _ = oracle.warp_bwd(vol, fld, gout)
    a, b = _gin_twice(dev(vol), dev(fld), dev(gout))
    assert np.array_equal(a, b)
    m = np.abs(want).max()
    assert rel_close(a / m, want / m, atol=1e-6), np.abs(a - want).max() / m


def test_warp_gin_fixed_point_nonfinite_channel(cuda, oracle, deterministic):
    """A channel whose upstream gradient holds NaN / Inf has no fixed-point
    scale: it is scattered in fp32 (NaN and Inf land where the reference puts
    them), the finite channels stay fixed point and repeatable."""
    dims = (24, 10, 9)
    vol = random_feature_map(3, dims, 18)
    fld = random_field(dims, 19, 1.2)
    gout = random_feature_map(3, dims, 20)
    gout[1, 4, 5, 6] = np.nan
    gout[2, 2, 3, 4] = np.inf
    want, _ = oracle.warp_bwd(vol, fld, gout)
    a, b = _gin_twice(dev(vol), dev(fld), dev(gout))
    assert np.array_equal(np.isnan(a), np.isnan(want))
    assert np.array_equal(np.isinf(a), np.isinf(want))
    fin = np.isfinite(want)
    assert rel_close(a[fin], want[fin])
    assert np.array_equal(a[0], b[0])


def test_compose_gprev_fixed_point_repeatable(cuda, oracle, deterministic):
    """Compose backward in deterministic mode: gprev (the scatter) by the
    fixed-point path, repeatable and within tolerance; gres bit-exact."""
    dims = (29, 17, 13)
    prev = random_field(dims, 21, 1.5)
    res = random_field(dims, 22, 2.5)
    gout = random_field(dims, 23, 1.0)
    wp, wr = oracle.compose_bwd(prev, res, gout)
    gp1, gr1 = ops.compose_bwd(dev(prev), dev(res), dev(gout))
    gp2, _ = ops.compose_bwd(dev(prev), dev(res), dev(gout))
    assert rel_close(host(gp1), wp)
    assert np.array_equal(host(gp1), host(gp2))
    assert np.array_equal(host(gr1), wr)


def test_warp_gin_gather_range_matches_whole(cuda, oracle, deterministic):
    """The voxel-range form (depth slabs / pipeline chunks) gathers the same
    terms: the sum over two ranges equals the whole-volume gradient."""
    dims = (32, 12, 20)
    vol = random_feature_map(2, dims, 7)
    fld = random_field(dims, 8, 1.7)
    gout = random_feature_map(2, dims, 9)
    from paper_2403_16526_b200 import _capi
    L = _capi.lib()
    n = 32 * 12 * 20
    whole, _ = ops.warp_bwd(dev(vol), dev(fld), dev(gout))
    gin = torch.zeros(2, n, device="cuda")
    v, f, g = dev(vol), dev(fld), dev(gout)
    for pb, pe in ((0, n // 3), (n // 3, n)):
        assert L.mdg_warp_bwd_range(v.data_ptr(), 2, ops.dims3(dims), f.data_ptr(), g.data_ptr(),
                                    gin.data_ptr(), None, pb, pe,
                                    torch.cuda.current_stream().cuda_stream) == 0
    assert rel_close(host(gin), host(whole).reshape(2, n))
