"""Maximum sizes: volumes whose channel-plane offsets exceed 2^31 elements
(64-bit offset paths, the 32-bit-offset gather's guard) checked through
size-independent properties with closed forms (no oracle at this size):

* warp fwd / bwd at 2^30 voxels with the constant field (1, 0, 0): the
  sample of voxel x is voxel x+1 exactly (clamped at the last column), the
  scatter moves every upstream gradient one voxel up, gfield_x is the exact
  forward difference (sampling.hpp:53-118);
* the ModeT operator at 2^28 voxels with K = 0, B = 0: uniform 1/27 weights
  (the reference's out-of-bounds rule gives the same logit), SF = 0 exactly,
  LSE = ln 27, dQ = 0 exactly, and dK in closed form on an interior block
  (attention.hpp:83-166)."""
import math

import pytest
import torch

from paper_2403_16526_b200 import ops

pytestmark = pytest.mark.gpu


def _free_gib():
    free, _ = torch.cuda.mem_get_info()
    return free / 2 ** 30


def test_warp_at_2_pow_30_voxels(cuda):
    if _free_gib() < 80:
        pytest.skip("needs ~70 GiB of free device memory")
    h = w = l = 1024  # 2^30 voxels: the field's z plane starts at 2^31 elements
    g = torch.Generator(device="cuda").manual_seed(3)
    vol = torch.rand(1, l, w, h, device="cuda", generator=g)
    field = torch.zeros(3, l, w, h, device="cuda")
    field[0] = 1.0
    out = ops.warp(vol, field)
    assert torch.equal(out[..., :-1], vol[..., 1:])
    assert torch.equal(out[..., -1], vol[..., -1])
    del out
    gout = torch.rand(1, l, w, h, device="cuda", generator=g)
    gin, gfield = ops.warp_bwd(vol, field, gout)
    # voxel x puts weight 1 on x+1 (x <= h-3), the last two columns on h-1
    assert not gin[..., 0].any()
    assert torch.equal(gin[..., 1:-1], gout[..., :-2])
    assert torch.equal(gin[..., -1], gout[..., -2] + gout[..., -1])
    # gfield_x where the x axis is live (0 < x+1 < h-1): g * (in[x+2] - in[x+1])
    exp_x = gout[0, :, :, :h - 2] * (vol[0, :, :, 2:] - vol[0, :, :, 1:h - 1])
    assert torch.equal(gfield[0, :, :, :h - 2], exp_x)
    assert torch.isfinite(gfield).all()


def test_modet_at_2_pow_28_voxels(cuda):
    if _free_gib() < 60:
        pytest.skip("needs ~50 GiB of free device memory")
    h, w, l = 512, 512, 1024  # 2^28 voxels; Q/K planes span 6 * 2^28 elements
    S, d = 1, 6
    cfg = ops.AttentionConfig(S, d, 3)
    n = h * w * l
    g = torch.Generator(device="cuda").manual_seed(5)
    Q = torch.rand(S * d, n, device="cuda", generator=g) * 2 - 1
    K = torch.zeros(S * d, n, device="cuda")
    B = torch.zeros(S, 27, device="cuda")
    SF, LSE = ops.modet_fwd(Q, K, B, (h, w, l), cfg, layout=ops.MDG_QK_PLANAR)
    assert not SF.any()  # uniform weights: the offsets cancel exactly
    assert torch.allclose(LSE, torch.full_like(LSE, math.log(27.0)), rtol=0, atol=2e-6)
    gSF = torch.rand(3 * S, n, device="cuda", generator=g) * 2 - 1
    gQ, gK, gB = ops.modet_bwd(Q, K, B, SF, LSE, gSF, (h, w, l), cfg, layout=ops.MDG_QK_PLANAR)
    assert not gQ.any()  # dQ = sum dl * K = 0
    assert torch.isfinite(gK).all() and torch.isfinite(gB).all()
    # dK_q = (1/27) sum_o (gSF_r . off(o)) Q_r, r = q - off(o) (SF = 0), on an
    # interior block of planes
    z0, z1 = 500, 504
    Qv, gv = Q.view(d, l, w, h), gSF.view(3, l, w, h)
    exp = torch.zeros(d, z1 - z0, w - 2, h - 2, device="cuda", dtype=torch.float64)
    for o in range(27):
        ox, oy, oz = o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1
        # sources r = q - off(o) for the keys q in [z0, z1) x [1, w-1) x [1, h-1)
        sl = (slice(z0 - oz, z1 - oz), slice(1 - oy, w - 1 - oy), slice(1 - ox, h - 1 - ox))
        dot = ox * gv[0][sl].double() + oy * gv[1][sl].double() + oz * gv[2][sl].double()
        exp += (dot / 27.0)[None] * Qv[(slice(None),) + sl].double()
    got = gK.view(d, l, w, h)[:, z0:z1, 1:w - 1, 1:h - 1].double()
    assert torch.allclose(got, exp, rtol=1e-4, atol=1e-5)
