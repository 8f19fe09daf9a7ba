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


def rel_norm(a, b):
    """||a - b|| / ||b|| (the per-tensor gradient criterion)."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def halved(d):
    """common.hpp:70-74 (ceil)."""
    return tuple((int(v) + 1) // 2 for v in d)


def pyramid_dims(fine, levels):
    """Level grids coarse -> fine as the encoder's avg-pool chain makes them."""
    ds = [tuple(fine)]
    for _ in range(levels - 1):
        ds.append(halved(ds[-1]))
    return ds[::-1]


def decoder_case(fine, levels, channels, heads, hd, seed, wscale=0.3):
    """Random features + packed level parameters (ModelParams::all_tensors
    order, engine.hpp:127-131) for decoder-pyramid parity.  Larger-than-init
    weights so attention is far from uniform; the RegHead is scaled so each
    level's residual is a fraction of a voxel (the regime registration runs in —
    with multi-voxel residuals on white-noise features the pyramid is chaotic
    and fp32 rounding differences grow without bound)."""
    r = np.random.default_rng(seed)
    dims = pyramid_dims(fine, levels)
    f_feats, m_feats, params = [], [], []
    for k, d in enumerate(dims):
        h, w, l = d
        C, S = channels[k], heads[k]
        K = S * hd
        f_feats.append(f32(r.standard_normal((C, l, w, h))))
        m_feats.append(f32(r.standard_normal((C, l, w, h))))
        blk = [r.standard_normal((K, C)) * wscale, r.standard_normal(K) * 0.1,
               r.uniform(0.5, 1.5, K), r.standard_normal(K) * 0.2,
               r.standard_normal((S, 27)) * 0.5,
               r.standard_normal((3, 3 * S, 3, 3, 3)) * (0.3 / np.sqrt(81 * S)),
               r.standard_normal(3) * 0.02]
        params.append(f32(np.concatenate([np.ravel(x) for x in blk])))
    return dims, f_feats, m_feats, params


def split_level_params(packed, C, S, hd):
    """Inverse of the packing: [proj_w, proj_b, ln_g, ln_b, rel_bias, rh_w, rh_b]."""
    K = S * hd
    sizes = [(K, C), (K,), (K,), (K,), (S, 27), (3, 3 * S, 3, 3, 3), (3,)]
    out, o = [], 0
    for s in sizes:
        m = int(np.prod(s))
        out.append(packed[o:o + m].reshape(s))
        o += m
    assert o == packed.size
    return out
