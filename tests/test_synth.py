"""The native synthetic-input generators (csrc/synth.cu) against the
reference: make_smooth_velocity and make_synth_pair (synth.cpp, through
oracle/_ref) bit for bit, and random_field (tests/test_util.hpp:40-48)
against a numpy restatement over the reference Rng stream."""
import numpy as np
import pytest
import torch

import pyoracle
from paper_2403_16526_b200 import ops


@pytest.mark.parametrize("dims,seed,mag,sigma", [((9, 8, 7), 11, 2.0, 4.0),
                                                 ((20, 12, 17), 3, 1.5, 1.2),
                                                 ((33, 5, 2), 7, 3.0, 0.0)])
def test_smooth_velocity_bit_exact(ref, dims, seed, mag, sigma):
    got = ops.make_smooth_velocity(dims, seed, mag, sigma).numpy()
    want = ref.make_smooth_velocity(dims, seed, mag, sigma)
    assert np.array_equal(got, want)


def test_random_field_matches_reference_stream():
    dims, seed, mag = (7, 6, 5), 13, 2.0
    got = ops.random_field(dims, seed, mag).numpy().ravel()
    u = pyoracle.Rng(seed).uniform01(2 * got.size).reshape(-1, 2)
    m = (0.15 + (1.0 - 0.15) * u[:, 0]) * mag
    want = np.where(u[:, 1] < 0.5, -m, m).astype(np.float32)
    assert np.array_equal(got, want)
    assert np.all(np.abs(got) >= 0.15 * mag * (1 - 1e-6)) and np.all(np.abs(got) <= mag)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,seed", [((32, 32, 32), 4), ((20, 16, 24), 9)])
def test_synth_pair_bit_exact(cuda, ref, dims, seed):
    f, m, lf, lm, gt = ops.synth_pair(dims, seed=seed, max_disp=2.0)
    rf, rm, rlf, rlm, rgt = ref.synth_pair(dims, seed=seed, max_disp=2.0)
    assert np.array_equal(m.numpy(), rm)
    assert np.array_equal(lm.numpy(), rlm)
    assert np.array_equal(gt.numpy(), rgt)
    assert np.array_equal(f.numpy(), rf)
    assert np.array_equal(lf.numpy(), rlf)
