"""GPU parity of the registration objective:
op_total_loss = NCC(fixed, warp(moving, phi)) + lambda * grad_reg(phi)
(objective.hpp:39-78, ops.hpp:301-382) against the REFERENCE's own tape
(oracle/_ref, ref_pipeline.cpp mdr_total_loss).

The warped image is bit-identical; the loss terms are means over the volume
(fixed-order tree vs the reference's sequential sum) and match to 1e-5
relative; gradients by relative norm <= 1e-4."""
import numpy as np
import pytest
import torch

from _util import f32, rel_norm
from paper_2403_16526_b200 import ops

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def smooth(dims, seed, amp):
    h, w, l = dims
    r = np.random.default_rng(seed)
    z, y, x = np.meshgrid(np.arange(l), np.arange(w), np.arange(h), indexing="ij")
    comps = []
    for c in range(3):
        a = r.uniform(0.5, 1.5, 3)
        ph = r.uniform(0, 6.28, 3)
        comps.append(amp * np.sin(x / (3 * a[0]) + ph[0]) * np.cos(y / (3 * a[1]) + ph[1])
                     * np.sin(z / (3 * a[2]) + ph[2]))
    return f32(np.stack(comps))


@pytest.mark.parametrize("dims,window,lam", [((12, 10, 8), 9, 1.0), ((9, 7, 11), 5, 0.5),
                                             ((17, 13, 6), 3, 0.0), ((20, 18, 16), 9, 1.0)])
def test_total_loss_matches_reference(cuda, ref, dims, window, lam):
    h, w, l = dims
    r = np.random.default_rng(sum(dims) + window)
    fixed = f32(r.uniform(0, 1, (1, l, w, h)))
    moving = f32(0.7 * fixed + 0.3 * r.uniform(0, 1, (1, l, w, h)))
    phi = smooth(dims, 3, 1.5)
    terms_r, warped_r, gphi_r, gm_r = ref.total_loss(fixed, moving, phi, window, lam)
    cfg = ops.LossConfig(lam=lam, ncc_window=window)
    terms, warped = ops.total_loss(dev(fixed), dev(moving), dev(phi), cfg, want_warped=True)
    assert np.array_equal(host(warped), warped_r)
    t = host(terms)
    assert np.allclose(t[:2], terms_r[:2], rtol=1e-5, atol=1e-7), (t, terms_r)
    if lam:
        assert np.allclose(t[2], terms_r[2], rtol=1e-5, atol=1e-9), (t, terms_r)
    gphi, gm = ops.total_loss_bwd(dev(fixed), dev(moving), dev(phi), cfg)
    assert rel_norm(host(gphi), gphi_r) <= 1e-4, rel_norm(host(gphi), gphi_r)
    assert rel_norm(host(gm), gm_r) <= 1e-4, rel_norm(host(gm), gm_r)


def test_perfect_match_scores_minus_one(cuda):
    """objective.hpp:36-37: a perfect match scores -1 up to the epsilon guard."""
    r = np.random.default_rng(0)
    img = f32(r.uniform(0, 1, (1, 10, 11, 12)))
    phi = np.zeros((3, 10, 11, 12), np.float32)
    t = host(ops.total_loss(dev(img), dev(img), dev(phi), ops.LossConfig(lam=1.0)))
    assert abs(t[1] + 1.0) < 1e-3 and t[2] == 0.0 and t[0] == t[1]


def test_loss_errors(cuda):
    img = dev(np.zeros((1, 4, 4, 4), np.float32))
    phi = dev(np.zeros((3, 4, 4, 4), np.float32))
    with pytest.raises(ops.InvalidInput, match="window"):
        ops.total_loss(img, img, phi, ops.LossConfig(ncc_window=4))
    with pytest.raises(ops.InvalidInput, match="lambda"):
        ops.total_loss(img, img, phi, ops.LossConfig(lam=-1.0))
