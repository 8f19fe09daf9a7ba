"""Scaling and squaring on the GPU against the reference's known-answer
properties (test_reghead.cpp:120-198): zero and constant velocities are exact,
T = 7 matches dense forward-Euler integration, small velocities integrate
fold-free, forward and backward integrations are mutually inverse, and the
result converges in T.  Velocities come from the reference's own
make_smooth_velocity (synth.cpp:75-90)."""
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
