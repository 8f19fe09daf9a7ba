"""Shared test helpers: seeded inputs identical to the reference test fixtures
(tests/test_util.hpp:24-48, test_attention.cpp:26-31), built on the oracle's
bit-identical Rng.  Test infrastructure only."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import pyoracle  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def random_qk(dims, sd, seed):
    """test_attention.cpp:26-31: {n, sd} N(0,1)."""
    h, w, l = dims
    return f32(pyoracle.Rng(seed).normal(h * w * l * sd).reshape(h * w * l, sd))


def random_volume(dims, seed, lo=0.0, hi=1.0, channels=1):
    """test_util.hpp:24-29 (uniform)."""
    h, w, l = dims
    return f32(pyoracle.Rng(seed).uniform(channels * h * w * l, lo, hi).reshape(channels, l, w, h))


def random_feature_map(c, dims, seed):
    """test_util.hpp:31-36 (normal)."""
    h, w, l = dims
    return f32(pyoracle.Rng(seed).normal(c * h * w * l).reshape(c, l, w, h))


def random_field(dims, seed, mag):
    """test_util.hpp:40-48: |entries| in [0.15, 1]*mag, random sign — consumed
    in the reference's interleaved order (magnitude draw, then sign draw)."""
    h, w, l = dims
    n3 = 3 * h * w * l
    u = pyoracle.Rng(seed).uniform01(2 * n3)
    m = (0.15 + (1.0 - 0.15) * u[0::2]) * mag
    v = np.where(u[1::2] < 0.5, -m, m)
    return f32(v.reshape(3, l, w, h))


def rel_close(a, b, atol=1e-5, rtol=1e-4):
    """North-star tolerance: |a-b| <= atol + rtol*|b| elementwise."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= atol + rtol * np.abs(b)))


def worst(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))
