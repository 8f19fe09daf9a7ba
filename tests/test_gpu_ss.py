"""Known-answer properties of the field operators on the GPU, restated from
the reference's tests.

Scaling and squaring (test_reghead.cpp:120-198): zero and constant velocities
are exact, T = 7 matches dense forward-Euler integration, small velocities
integrate fold-free, forward and backward integrations are mutually inverse,
and the result converges in T (velocities from the reference's
make_smooth_velocity, synth.cpp:75-90).  Compose (test_field_ops.cpp:112-160):
zero is the identity, constants add, warping by a composite matches
sequential warps, and composition is associative (the reference's own
smooth_field / smooth_image test data)."""
import numpy as np
import pytest
import torch

from paper_2403_16526_b200 import ops

pytestmark = pytest.mark.gpu


def smooth(ref, dims, seed, mag, sigma):
    return torch.from_numpy(ref.make_smooth_velocity(dims, seed, mag, sigma)).cuda()


def jacobian_det(phi):
    """field_ops.hpp:52-84: det(I + grad u), central differences inside,
    one-sided at the borders (np.gradient's first-order edges)."""
    u = phi.cpu().numpy().astype(np.float32)  # {3, l, w, h}
    # axis order of u[comp]: (z, y, x); reference axes: 0 = x, 1 = y, 2 = z
    grads = [[np.gradient(u[c], axis=2 - a) for a in range(3)] for c in range(3)]
    m = [[grads[c][a] + (1.0 if c == a else 0.0) for a in range(3)] for c in range(3)]
    return (m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1])
            - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0])
            + m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]))


def test_ss_zero_and_constant_exact(cuda):
    v = torch.zeros(3, 5, 5, 5, device="cuda")
    for steps in (1, 4, 7):
        assert bool((ops.scaling_squaring(v, steps) == 0).all())
    c = torch.zeros(3, 6, 4, 5, device="cuda")
    c[0] = 0.8125
    c[1] = -0.25
    for steps in (1, 3, 7):
        phi = ops.scaling_squaring(c, steps)
        assert bool((phi == c).all())


def test_ss_matches_dense_euler(cuda, ref):
    dims = (12, 12, 12)
    v = smooth(ref, dims, 11, 0.5, 4.0)
    ss = ops.scaling_squaring(v, 7)
    phi = torch.zeros_like(v)
    hstep = np.float32(1.0 / 128)
    for _ in range(128):  # d phi / dt = v(x + phi), forward Euler
        phi = phi + hstep * ops.warp(v, phi)
    assert float((ss - phi).abs().max()) <= 1e-3


def test_ss_small_velocities_fold_free(cuda, ref):
    for seed in range(1, 6):
        phi = ops.scaling_squaring(smooth(ref, (10, 10, 10), seed, 0.4, 2.0), 7)
        assert float((jacobian_det(phi) <= 0).mean()) == 0.0


def test_ss_forward_backward_inverse(cuda, ref):
    v = smooth(ref, (10, 10, 10), 17, 0.3, 4.0)
    fwd = ops.scaling_squaring(v, 7)
    bwd = ops.scaling_squaring(-v, 7)
    assert float(ops.compose(fwd, bwd).abs().max()) <= 1e-2


def test_ss_converges_in_steps(cuda, ref):
    v = smooth(ref, (10, 10, 10), 19, 0.4, 4.0)
    a = ops.scaling_squaring(v, 7)
    b = ops.scaling_squaring(v, 8)
    assert float((a - b).abs().max()) <= 1e-3


# ---- compose known answers (test_field_ops.cpp:112-160)
def test_compose_identity_and_constants(cuda):
    g = torch.Generator().manual_seed(11)
    f = (torch.rand(3, 5, 5, 5, generator=g) * 2 - 1).cuda()
    zero = torch.zeros_like(f)
    assert torch.allclose(ops.compose(f, zero), f, rtol=1e-6, atol=0)
    assert torch.allclose(ops.compose(zero, f), f, rtol=1e-6, atol=1e-7)
    a = torch.zeros(3, 4, 4, 4, device="cuda")
    b = torch.zeros_like(a)
    a[0], a[2] = 0.4, -0.2
    b[0], b[1] = 0.3, 0.1
    c = ops.compose(a, b)
    for comp, want in ((0, 0.7), (1, 0.1), (2, -0.2)):
        assert torch.allclose(c[comp], torch.full_like(c[comp], want), rtol=1e-6, atol=0)


def _rng_draws(seed, specs):
    r = ops.Rng(seed)
    return [float(r.uniform((1,), lo, hi)[0]) for lo, hi in specs]


def _smooth_field(dims, amplitude, waves, seed):
    """test_field_ops.cpp:15-34 smooth_field (the reference's test data)."""
    h, w, l = dims
    z, y, x = np.meshgrid(np.arange(l), np.arange(w), np.arange(h), indexing="ij")
    r = ops.Rng(seed)
    out = np.zeros((3, l, w, h), np.float32)
    tp = np.float32(2.0 * 3.14159265)
    for comp in range(3):
        ax, px, py, pz = (float(r.uniform((1,), lo, hi)[0])
                          for lo, hi in ((0.2, 1.0), (0.0, 6.28), (0.0, 6.28), (0.0, 6.28)))
        out[comp] = (np.float32(amplitude) * np.float32(ax)
                     * np.sin(tp * x / np.float32(waves * h) + np.float32(px))
                     * np.cos(tp * y / np.float32(waves * w) + np.float32(py))
                     * np.sin(tp * z / np.float32(waves * l) + np.float32(pz))).astype(np.float32)
    return torch.from_numpy(out).cuda()


def _smooth_image(dims, waves, seed):
    """test_field_ops.cpp:36-48 smooth_image."""
    h, w, l = dims
    z, y, x = np.meshgrid(np.arange(l), np.arange(w), np.arange(h), indexing="ij")
    p1, p2 = _rng_draws(seed, ((0.0, 6.28), (0.0, 6.28)))
    tp = np.float32(2.0 * 3.14159265)
    v = np.float32(0.6) * (np.sin(tp * x / np.float32(waves * h) + np.float32(p1))
                           * np.cos(tp * (y + z) / np.float32(waves * (w + l)) + np.float32(p2))
                           + np.float32(0.5) * np.cos(tp * z / np.float32(waves * l)
                                                      + np.float32(p1)))
    return torch.from_numpy(v.astype(np.float32)).cuda().view(1, l, w, h).contiguous()


def test_compose_matches_sequential_warps(cuda):
    dims = (8, 8, 8)
    img = _smooth_image(dims, 2.5, 13)
    prev = _smooth_field(dims, 0.8, 2.5, 17)
    res = _smooth_field(dims, 0.8, 2.5, 19)
    once = ops.warp(img, ops.compose(prev, res))
    twice = ops.warp(ops.warp(img, prev), res)
    assert float((once - twice).abs().max()) <= 2e-2


def test_compose_associative(cuda):
    dims = (8, 8, 8)
    a, b, c = (_smooth_field(dims, 0.9, 3.5, s) for s in (23, 29, 31))
    left = ops.compose(ops.compose(a, b), c)
    right = ops.compose(a, ops.compose(b, c))
    assert float((left - right).abs().max()) <= 5e-2
