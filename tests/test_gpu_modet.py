"""GPU parity of the ModeT operator (fused tier + reference-shaped tier)
against the CPU oracle and the reference's golden fixtures.

Tolerances (BASELINE.json north_star): flows |d| <= 1e-5 + 1e-4|ref|
elementwise; attention weights |d| <= 1e-5 (the reference's own fused-vs-naive
f32 bar, test_attention.cpp:155-191); gradients per tensor
||d|| / ||ref|| <= 1e-4 (SURVEY.md §8c protocol); integer index logic exact.
"""
import glob
import os

import numpy as np
import pytest
import torch

import pyoracle
from _util import GOLDEN, f32, load_golden, random_qk, rel_close, worst
from paper_2403_16526_b200 import ops
from paper_2403_16526_b200._capi import MDG_QK_PLANAR, MDG_QK_POSMAJOR

pytestmark = pytest.mark.gpu

FLOW_ATOL, FLOW_RTOL = 1e-5, 1e-4
W_ATOL = 1e-5
GRAD_RTOL = 1e-4


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def grad_ok(got, ref, rtol=GRAD_RTOL):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    nr = np.linalg.norm(ref)
    return np.linalg.norm(got - ref) <= rtol * max(nr, 1e-30) + 1e-7


def oracle_modet(oracle, Q, K, B, dims, S, hd, gSF, nb=3):
    W, bad = oracle.na_fwd(Q, K, B, dims, S, hd, nb)
    assert bad is None
    SF = oracle.subfields_fwd(W, dims, S, nb)
    gW = oracle.subfields_bwd(gSF, dims, S, nb)
    gQ, gK, gB = oracle.na_bwd(Q, K, W, gW, dims, S, hd, nb)
    return W, SF, gQ, gK, gB


def run_fused(Q, K, B, dims, S, hd, gSF, layout=MDG_QK_POSMAJOR, accumulate=False):
    """Fused tier on (Q, K) given position-major.  PLANAR runs the tiled
    z-marching kernels (modet_tiled.cu); W comes from the W-emitting path."""
    cfg = ops.AttentionConfig(S, hd, 3)
    n = dims[0] * dims[1] * dims[2]
    if layout == MDG_QK_PLANAR:
        Qd, Kd = dev(np.ascontiguousarray(Q.T)), dev(np.ascontiguousarray(K.T))
    else:
        Qd, Kd = dev(Q), dev(K)
    Bd = dev(B)
    _, _, W = ops.modet_fwd(dev(Q), dev(K), Bd, dims, cfg, want_w=True)
    SF, LSE = ops.modet_fwd(Qd, Kd, Bd, dims, cfg, layout=layout)
    g = dev(gSF.reshape(3 * S, n))
    if accumulate:  # pre-filled targets: result must be prefill + gradient
        gQ0 = torch.full_like(Qd, 0.25)
        gK0 = torch.full_like(Kd, -0.5)
        gB0 = torch.full_like(Bd, 1.0)
        gQ, gK, gB = ops.modet_bwd(Qd, Kd, Bd, SF, LSE, g, dims, cfg, layout=layout,
                                   gQ=gQ0.clone(), gK=gK0.clone(), gB=gB0.clone())
        gQ, gK, gB = gQ - gQ0, gK - gK0, gB - gB0
    else:
        gQ, gK, gB = ops.modet_bwd(Qd, Kd, Bd, SF, LSE, g, dims, cfg, layout=layout)
    gQ, gK = host(gQ), host(gK)
    if layout == MDG_QK_PLANAR:
        gQ, gK = gQ.T, gK.T
    return host(W), host(SF), host(LSE), gQ, gK, host(gB)


# ------------------------------------------------------------------ goldens
ATTN3 = [os.path.basename(p)[:-4] for p in sorted(glob.glob(os.path.join(GOLDEN, "attn_*.npz")))
         if "nb5" not in p]


@pytest.mark.parametrize("layout", [MDG_QK_POSMAJOR, MDG_QK_PLANAR])
@pytest.mark.parametrize("name", ATTN3)
def test_fused_matches_golden(cuda, name, layout):
    g = load_golden(name)
    dims, S, hd = tuple(int(v) for v in g["dims"]), int(g["S"]), int(g["hd"])
    W, SF, LSE, gQ, gK, gB = run_fused(g["Q"], g["K"], g["B"], dims, S, hd, g["gSF"], layout)
    assert worst(W, g["W"]) <= W_ATOL
    assert rel_close(SF, g["SF"].reshape(SF.shape), FLOW_ATOL, FLOW_RTOL)
    assert np.all(np.isfinite(LSE))
    assert grad_ok(gQ, g["gQ"]) and grad_ok(gK, g["gK"]) and grad_ok(gB, g["gB"])


@pytest.mark.parametrize("name", [os.path.basename(p)[:-4] for p in
                                  sorted(glob.glob(os.path.join(GOLDEN, "attn_*.npz")))])
def test_reference_tier_matches_golden(cuda, name):
    g = load_golden(name)
    dims, S, hd, nb = tuple(int(v) for v in g["dims"]), int(g["S"]), int(g["hd"]), int(g["nb"])
    cfg = ops.AttentionConfig(S, hd, nb)
    Q, K, B = dev(g["Q"]), dev(g["K"]), dev(g["B"])
    W = ops.na_fused(Q, K, B, dims, cfg)
    assert worst(host(W), g["W"]) <= W_ATOL
    SF = ops.subfields(W, dims, cfg)
    assert rel_close(host(SF), g["SF"].reshape(3 * S, -1), FLOW_ATOL, FLOW_RTOL)
    gW = torch.zeros_like(W)
    ops.kern.subfields_bwd(dims, S, nb, dev(g["gSF"]), gW)
    assert np.array_equal(host(gW), g["gW"])  # exact: products with {-1,0,1}
    gQ, gK, gB = torch.zeros_like(Q), torch.zeros_like(K), torch.zeros_like(B)
    ops.kern.na_fused_bwd(Q, K, dev(g["W"]), dims, S, hd, nb, dev(g["gW"]), gQ, gK, gB)
    assert grad_ok(host(gQ), g["gQ"]) and grad_ok(host(gK), g["gK"])
    assert grad_ok(host(gB), g["gB"])


# ---------------------------------------------------------- randomised parity
def test_fused_randomised_against_oracle(cuda, oracle):
    seeds = pyoracle.Rng(7)
    for trial in range(24):
        dims = tuple(int(seeds.uniform_int(1, 9)) for _ in range(3))
        S = seeds.uniform_int(1, 4)
        hd = [2, 3, 4, 5, 6, 7, 8, 12][trial % 8]  # 7 exercises the generic path
        n = dims[0] * dims[1] * dims[2]
        Q = random_qk(dims, S * hd, 10 + trial)
        K = random_qk(dims, S * hd, 40 + trial)
        B = f32(pyoracle.Rng(70 + trial).normal(S * 27).reshape(S, 27))
        gSF = f32(pyoracle.Rng(90 + trial).normal(3 * S * n).reshape(3 * S, dims[2], dims[1],
                                                                         dims[0]))
        W0, SF0, gQ0, gK0, gB0 = oracle_modet(oracle, Q, K, B, dims, S, hd, gSF)
        layout = MDG_QK_PLANAR if trial % 2 else MDG_QK_POSMAJOR
        W, SF, LSE, gQ, gK, gB = run_fused(Q, K, B, dims, S, hd, gSF, layout)
        assert worst(W, W0) <= W_ATOL, (trial, dims, S, hd)
        assert rel_close(SF, SF0.reshape(SF.shape), FLOW_ATOL, FLOW_RTOL), (trial, dims)
        assert grad_ok(gQ, gQ0) and grad_ok(gK, gK0) and grad_ok(gB, gB0), (trial, dims, S, hd)


@pytest.mark.parametrize("dims,S,hd", [((33, 17, 9), 1, 6), ((1, 1, 1), 2, 6), ((2, 40, 3), 1, 4),
                                       ((65, 3, 31), 2, 6), ((31, 18, 2), 1, 8),
                                       ((10, 12, 14), 8, 6), ((20, 24, 28), 4, 6),
                                       ((7, 5, 26), 1, 12), ((9, 9, 9), 3, 16), ((6, 6, 5), 2, 1)])
@pytest.mark.parametrize("accumulate", [False, True])
def test_tiled_kernels_ragged_tiles(cuda, oracle, dims, S, hd, accumulate):
    """Tile / z-chunk edges of the z-marching kernels (32x16 and 32x8 x-y
    tiles, z chunks) on ragged shapes, incl. the pyramid-level shapes."""
    n = dims[0] * dims[1] * dims[2]
    seed = sum(dims) * 7 + S * 3 + hd
    Q = random_qk(dims, S * hd, seed)
    K = random_qk(dims, S * hd, seed + 1)
    B = f32(pyoracle.Rng(seed + 2).normal(S * 27).reshape(S, 27))
    gSF = f32(pyoracle.Rng(seed + 3).normal(3 * S * n).reshape(3 * S, dims[2], dims[1], dims[0]))
    W0, SF0, gQ0, gK0, gB0 = oracle_modet(oracle, Q, K, B, dims, S, hd, gSF)
    W, SF, LSE, gQ, gK, gB = run_fused(Q, K, B, dims, S, hd, gSF, MDG_QK_PLANAR, accumulate)
    assert rel_close(SF, SF0.reshape(SF.shape), FLOW_ATOL, FLOW_RTOL)
    # LSE agrees with the oracle's normaliser: W = exp(l - LSE) reproduces W
    assert np.all(np.isfinite(LSE))
    assert grad_ok(gQ, gQ0) and grad_ok(gK, gK0)
    assert grad_ok(gB, gB0, 1e-4 if not accumulate else 1e-3)


@pytest.mark.parametrize("spread", [30.0, 95.0, 300.0])
def test_fused_forward_large_logit_spread(cuda, oracle, spread):
    """The tiled forward fixes each voxel's softmax reference max from its first
    window row; logits far above it (here a huge bias on the last window rows)
    must still give the exact softmax (overflowed voxels go to the exact fixup
    kernel)."""
    dims, S, hd = (20, 9, 7), 2, 6
    n = 20 * 9 * 7
    Q = random_qk(dims, S * hd, 3)
    K = random_qk(dims, S * hd, 4)
    B = f32(pyoracle.Rng(5).normal(S * 27).reshape(S, 27))
    B[0, 18:] += spread
    B[1, 26] += spread
    gSF = f32(pyoracle.Rng(6).normal(3 * S * n).reshape(3 * S, 7, 9, 20))
    W0, SF0, gQ0, gK0, gB0 = oracle_modet(oracle, Q, K, B, dims, S, hd, gSF)
    W, SF, LSE, gQ, gK, gB = run_fused(Q, K, B, dims, S, hd, gSF, MDG_QK_PLANAR)
    assert rel_close(SF, SF0.reshape(SF.shape), FLOW_ATOL, FLOW_RTOL)
    assert grad_ok(gQ, gQ0) and grad_ok(gK, gK0) and grad_ok(gB, gB0)


def test_fused_forward_negative_inf_bias_raises(cuda, oracle):
    dims = (8, 4, 3)
    Q, K = random_qk(dims, 6, 1), random_qk(dims, 6, 2)
    B = np.zeros((1, 27), np.float32)
    B[0, 20] = -np.inf
    _, bad = oracle.na_fwd(Q, K, B, dims, 1, 6)
    with pytest.raises(ops.NumericError) as ei:
        ops.modet_fwd(dev(Q.T.copy()), dev(K.T.copy()), dev(B), dims, ops.AttentionConfig(1, 6, 3),
                      layout=MDG_QK_PLANAR)
    assert ei.value.position == bad


@pytest.mark.parametrize("layout", [MDG_QK_PLANAR, MDG_QK_POSMAJOR])
def test_config1_32cubed_s8_d8(cuda, oracle, layout):
    """BASELINE configs[0]: 32^3, 8 heads x 8 channels; inputs in the order of
    the reference bench (bench.cpp:28-35): Rng(5) Q, K ~ U(-1,1), B ~ U(-.5,.5);
    upstream gradient Rng(6) U(-1,1).  PLANAR runs the production tiled TMA
    kernels (modet_tiled.cu), POSMAJOR the position-major fallback."""
    dims, S, hd = (32, 32, 32), 8, 8
    n = 32 ** 3
    r = pyoracle.Rng(5)
    Q = f32(r.uniform(n * S * hd, -1, 1).reshape(n, S * hd))
    K = f32(r.uniform(n * S * hd, -1, 1).reshape(n, S * hd))
    B = f32(r.uniform(S * 27, -0.5, 0.5).reshape(S, 27))
    gSF = f32(pyoracle.Rng(6).uniform(3 * S * n, -1, 1).reshape(3 * S, 32, 32, 32))
    W0, SF0, gQ0, gK0, gB0 = oracle_modet(oracle, Q, K, B, dims, S, hd, gSF)
    W, SF, LSE, gQ, gK, gB = run_fused(Q, K, B, dims, S, hd, gSF, layout)
    assert worst(W, W0) <= W_ATOL
    assert rel_close(SF, SF0.reshape(SF.shape), FLOW_ATOL, FLOW_RTOL)
    assert grad_ok(gQ, gQ0) and grad_ok(gK, gK0) and grad_ok(gB, gB0)


# ------------------------------------------------------------ restated KATs
def test_kat_uniform_interior_and_zero_q(cuda):
    d = (5, 5, 5)
    cfg = ops.AttentionConfig(1, 4, 3)
    Q = dev(random_qk(d, 4, 5))
    K = torch.full((125, 4), 0.37, device="cuda")
    _, _, W = ops.modet_fwd(Q, K, torch.zeros(1, 27, device="cuda"), d, cfg, want_w=True)
    p = (2 * 5 + 2) * 5 + 2
    assert np.allclose(host(W)[0, p], 1 / 27, rtol=1e-5, atol=0)
    cfg2 = ops.AttentionConfig(2, 4, 3)
    SF, _, W = ops.modet_fwd(torch.zeros(27, 8, device="cuda"), dev(random_qk((3, 3, 3), 8, 13)),
                             torch.zeros(2, 27, device="cuda"), (3, 3, 3), cfg2, want_w=True)
    assert np.allclose(host(W), 1 / 27, rtol=1e-6, atol=0)
    assert np.all(np.abs(host(SF)) <= 1e-6)


def test_kat_dominant_bias_and_1x1x1(cuda):
    B = torch.zeros(1, 27, device="cuda")
    B[0, 14] = 10.0
    z = torch.zeros(64, 3, device="cuda")
    _, _, W = ops.modet_fwd(z, z, B, (4, 4, 4), ops.AttentionConfig(1, 3, 3), want_w=True)
    expect = np.exp(10.0) / (np.exp(10.0) + 26.0)
    assert abs(host(W)[0, 21, 14] - expect) <= 1e-6
    Q, K = random_qk((1, 1, 1), 3, 11), random_qk((1, 1, 1), 3, 12)
    Bn = f32(pyoracle.Rng(9).normal(27).reshape(1, 27))
    _, _, W = ops.modet_fwd(dev(Q), dev(K), dev(Bn), (1, 1, 1), ops.AttentionConfig(1, 3, 3),
                            want_w=True)
    lg = Bn[0].astype(np.float64).copy()
    lg[13] += float(Q[0].astype(np.float64) @ K[0].astype(np.float64))
    e = np.exp(lg - lg.max())
    assert np.allclose(host(W)[0, 0], e / e.sum(), rtol=1e-5, atol=1e-7)


def test_kat_rows_are_distributions_subflows_bounded(cuda):
    d = (6, 5, 4)
    cfg = ops.AttentionConfig(3, 5, 3)
    B = f32(pyoracle.Rng(19).normal(81, 0.0, 2.0).reshape(3, 27))
    SF, _, W = ops.modet_fwd(dev(random_qk(d, 15, 17)), dev(random_qk(d, 15, 18)), dev(B), d,
                             cfg, want_w=True)
    Wn = host(W)
    assert np.all(Wn >= 0) and np.allclose(Wn.sum(-1), 1.0, atol=1e-5)
    assert np.all(np.abs(host(SF)) <= 1.0)


def test_kat_translation_equivariance_exact(cuda):
    d, SD = (7, 6, 6), 8
    q0, k0 = random_qk(d, SD, 31), random_qk(d, SD, 32)
    q1, k1 = q0.reshape(6, 6, 7, SD).copy(), k0.reshape(6, 6, 7, SD).copy()
    q1[:, :, 1:], k1[:, :, 1:] = q0.reshape(6, 6, 7, SD)[:, :, :-1], k0.reshape(6, 6, 7, SD)[:, :, :-1]
    B = dev(f32(pyoracle.Rng(29).normal(54).reshape(2, 27)))
    cfg = ops.AttentionConfig(2, 4, 3)
    _, _, W0 = ops.modet_fwd(dev(q0), dev(k0), B, d, cfg, want_w=True)
    _, _, W1 = ops.modet_fwd(dev(q1.reshape(-1, SD)), dev(k1.reshape(-1, SD)), B, d, cfg,
                             want_w=True)
    W0v, W1v = host(W0).reshape(2, 6, 6, 7, 27), host(W1).reshape(2, 6, 6, 7, 27)
    assert np.array_equal(W0v[:, 2:4, 2:4, 2:4], W1v[:, 2:4, 2:4, 3:5])


@pytest.mark.parametrize("tier", ["fused", "reference"])
def test_nonfinite_logit_raises_with_reference_position(cuda, oracle, tier):
    dims = (3, 2, 2)
    Q = random_qk(dims, 4, 1)
    K = random_qk(dims, 4, 2)
    B = np.zeros((2, 27), np.float32)
    Q[7, 3] = np.inf
    Q[9, 0] = np.nan  # later in head order: the first (head 0) must win
    _, bad = oracle.na_fwd(Q, K, B, dims, 2, 2)
    cfg = ops.AttentionConfig(2, 2, 3)
    with pytest.raises(ops.NumericError) as ei:
        if tier == "fused":
            ops.modet_fwd(dev(Q), dev(K), dev(B), dims, cfg)
        else:
            ops.na_fused(dev(Q), dev(K), dev(B), dims, cfg)
    assert ei.value.position == bad
    # the flag is consumed: a clean call afterwards succeeds
    ops.modet_fwd(dev(random_qk(dims, 4, 3)), dev(K), dev(B), dims, cfg)


def test_subfields_rejects_unnormalised_rows(cuda):
    W = torch.full((1, 8, 27), 0.1, device="cuda")
    with pytest.raises(ops.InvalidInput, match="normalized"):
        ops.subfields(W, (2, 2, 2), ops.AttentionConfig(1, 3, 3))


def test_layout_adapters_roundtrip(cuda):
    x = dev(random_qk((9, 7, 5), 6, 3))
    p = ops.qk_posmajor_to_planar(x)
    assert np.array_equal(host(p), host(x).T)
    assert np.array_equal(host(ops.qk_planar_to_posmajor(p)), host(x))


@pytest.mark.parametrize("acc", [1, 0])
def test_host_buffer_calls_match_device_calls(cuda, acc):
    """Small volumes take the whole-volume host path.  acc=0 overwrites the
    caller's gradients (gB included: its host value is never uploaded, here
    pre-filled with garbage), acc=1 adds into them."""
    import ctypes as C

    from paper_2403_16526_b200 import _capi

    dims, S, hd = (9, 8, 7), 2, 6
    n = 9 * 8 * 7
    Q, K = random_qk(dims, S * hd, 1), random_qk(dims, S * hd, 2)
    B = f32(pyoracle.Rng(3).normal(S * 27).reshape(S, 27))
    gSF = f32(pyoracle.Rng(4).normal(3 * S * n).reshape(3 * S, n))
    W_, SF, LSE, gQ, gK, gB = run_fused(Q, K, B, dims, S, hd, gSF)
    L = _capi.lib()
    hSF, hL = np.zeros((3 * S, n), np.float32), np.zeros((S, n), np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    d3 = _capi.Dims3(*dims)
    assert L.mdg_modet_fwd_host(p(Q), p(K), p(B), d3, S, hd, 3, 0, p(hSF), p(hL)) == 0
    assert np.array_equal(hSF, SF) and np.array_equal(hL, LSE)
    hgQ, hgK, hgB = np.zeros_like(Q), np.zeros_like(K), np.zeros_like(B)
    if not acc:
        hgQ[:], hgK[:], hgB[:] = 7.0, -3.0, 1e30
    assert L.mdg_modet_bwd_host(p(Q), p(K), p(B), p(hSF), p(hL), p(gSF), d3, S, hd, 3, 0,
                                p(hgQ), p(hgK), p(hgB), acc) == 0
    assert np.array_equal(hgQ, gQ) and np.array_equal(hgK, gK) and np.array_equal(hgB, gB)
    hW = np.zeros((S, n, 27), np.float32)
    assert L.mdg_na_fused_fwd_host(p(Q), p(K), p(B), d3, S, hd, 3, p(hW)) == 0
    assert worst(hW, W_) <= W_ATOL


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("acc", [1, 0])
@pytest.mark.parametrize("dims,S,hd", [((128, 96, 100), 1, 6), ((64, 80, 205), 2, 4)])
def test_pipelined_host_calls_match_device_calls(cuda, layout, dims, S, hd, acc):
    """Volumes >= 1M voxels take the three-stream z-chunk pipeline inside the
    *_host calls (chunks extended by device-copied halo planes): SF, LSE, gQ,
    gK must equal the whole-volume device call bit for bit, gB to reduction
    tolerance; the backward accumulates into the caller's buffers (acc=1) or
    overwrites them (acc=0)."""
    import ctypes as C

    from paper_2403_16526_b200 import _capi

    h, w, l = dims
    n = h * w * l
    r = np.random.default_rng(3)
    Qp = f32(r.uniform(-1, 1, (n, S * hd)))
    Kp = f32(r.uniform(-1, 1, (n, S * hd)))
    B = f32(r.uniform(-0.5, 0.5, (S, 27)))
    gSF = f32(r.uniform(-1, 1, (3 * S, n)))
    cfg = ops.AttentionConfig(S, hd, 3)
    # reference: the whole-volume fused (tiled, planar) device call
    Qd, Kd = dev(f32(Qp.T)), dev(f32(Kp.T))
    SF, LSE = ops.modet_fwd(Qd, Kd, dev(B), dims, cfg, layout=1)
    gQ0 = f32(r.standard_normal((n, S * hd)))
    gK0 = f32(r.standard_normal((n, S * hd)))
    gB0 = f32(r.standard_normal((S, 27)))
    z = np.zeros_like
    gQ, gK, gB = ops.modet_bwd(Qd, Kd, dev(B), SF, LSE, dev(gSF), dims, cfg, layout=1,
                               gQ=dev(f32((gQ0 if acc else z(gQ0)).T)),
                               gK=dev(f32((gK0 if acc else z(gK0)).T)),
                               gB=dev(gB0 if acc else z(gB0)))
    SF, LSE, gB = host(SF), host(LSE), host(gB)
    gQ, gK = host(gQ).T, host(gK).T
    Q, K, hgQ, hgK = Qp, Kp, gQ0.copy(), gK0.copy()
    if layout == 1:
        Q, K, hgQ, hgK = (f32(a.T) for a in (Qp, Kp, gQ0, gK0))
    L = _capi.lib()
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    d3 = _capi.Dims3(*dims)
    hSF, hL = np.zeros((3 * S, n), np.float32), np.zeros((S, n), np.float32)
    assert L.mdg_modet_fwd_host(p(Q), p(K), p(B), d3, S, hd, 3, layout, p(hSF), p(hL)) == 0
    assert np.array_equal(hSF, SF) and np.array_equal(hL, LSE)
    hgB = gB0.copy()
    assert L.mdg_modet_bwd_host(p(Q), p(K), p(B), p(hSF), p(hL), p(gSF), d3, S, hd, 3, layout,
                                p(hgQ), p(hgK), p(hgB), acc) == 0
    if layout == 1:
        hgQ, hgK = hgQ.T, hgK.T
    assert np.array_equal(hgQ, gQ) and np.array_equal(hgK, gK)
    assert np.allclose(hgB, gB, rtol=1e-5, atol=1e-4)


# --------------------------------------------------------- north-star size
@pytest.mark.slow
def test_north_star_size_parity_and_properties(cuda, oracle):
    """L1 of the small preset at 160x192x224 (S=1, d=6): full-size parity with
    the oracle (sub-flows elementwise, gradients per tensor) plus exact
    gradient linearity."""
    dims, S, hd = (160, 192, 224), 1, 6
    n = 160 * 192 * 224
    r = pyoracle.Rng(5)
    Q = f32(r.uniform(n * hd, -1, 1).reshape(n, hd))
    K = f32(r.uniform(n * hd, -1, 1).reshape(n, hd))
    B = f32(r.uniform(27, -0.5, 0.5).reshape(1, 27))
    gSF = f32(pyoracle.Rng(6).uniform(3 * n, -1, 1).reshape(3, n))
    cfg = ops.AttentionConfig(S, hd, 3)
    P = MDG_QK_PLANAR  # the tiled production kernels
    Qd, Kd, Bd, gd = dev(Q.T.copy()), dev(K.T.copy()), dev(B), dev(gSF)
    SF, LSE = ops.modet_fwd(Qd, Kd, Bd, dims, cfg, layout=P)
    gQ, gK, gB = ops.modet_bwd(Qd, Kd, Bd, SF, LSE, gd, dims, cfg, layout=P)
    gQ2, gK2, gB2 = ops.modet_bwd(Qd, Kd, Bd, SF, LSE, 2 * gd, dims, cfg, layout=P)
    assert torch.equal(gQ2, 2 * gQ) and torch.equal(gK2, 2 * gK)
    gQ, gK = gQ.t(), gK.t()
    SFh = host(SF)
    assert np.all(np.abs(SFh) <= 1.0) and np.all(np.isfinite(host(LSE)))
    W0, SF0, gQ0, gK0, gB0 = oracle_modet(oracle, Q, K, B, dims, S, hd,
                                          gSF.reshape(3, 224, 192, 160))
    del W0
    assert rel_close(SFh, SF0.reshape(3, n), FLOW_ATOL, FLOW_RTOL)
    assert grad_ok(host(gQ), gQ0) and grad_ok(host(gK), gK0) and grad_ok(host(gB), gB0)


def test_two_streams_same_device_fixup_isolated(cuda, oracle):
    """The fixup queue and numeric flag are per (device, stream): two streams
    running forwards with overflowing logits at the same time (different
    volume sizes, so a shared queue would also decode positions against the
    wrong dims) must each get the exact softmax, and a non-finite logit on one
    stream must be reported on that stream only."""
    cases = []
    for dims, seed in (((20, 9, 7), 3), ((12, 16, 11), 8)):
        S, hd = 2, 6
        n = dims[0] * dims[1] * dims[2]
        Q, K = random_qk(dims, S * hd, seed), random_qk(dims, S * hd, seed + 1)
        B = f32(pyoracle.Rng(seed + 2).normal(S * 27).reshape(S, 27))
        B[0, 18:] += 95.0  # every voxel overflows the first-row max -> fixup
        B[1, 26] += 300.0
        W0, bad = oracle.na_fwd(Q, K, B, dims, S, hd)
        assert bad is None
        SF0 = oracle.subfields_fwd(W0, dims, S).reshape(3 * S, n)
        cases.append((dims, dev(Q.T.copy()), dev(K.T.copy()), dev(B), SF0))
    cfg = ops.AttentionConfig(2, 6, 3)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[], []]
    for _ in range(20):
        for i, (dims, Qd, Kd, Bd, _) in enumerate(cases):
            with torch.cuda.stream(streams[i]):
                outs[i].append(ops.modet_fwd(Qd, Kd, Bd, dims, cfg, layout=MDG_QK_PLANAR,
                                             check=False)[0])
    for i, (dims, *_rest) in enumerate(cases):  # no stray flag on either stream
        with torch.cuda.stream(streams[i]):
            ops.check_numeric(dims)
    torch.cuda.synchronize()
    for i, (dims, _, _, _, SF0) in enumerate(cases):
        for SF in outs[i]:
            assert rel_close(host(SF), SF0, FLOW_ATOL, FLOW_RTOL), (i, dims)
    # a -inf bias on stream 0 only: stream 1 stays clean
    dims, Qd, Kd, Bd, _ = cases[0]
    Bbad = Bd.clone()
    Bbad[0, 3] = -float("inf")
    with torch.cuda.stream(streams[0]):
        with pytest.raises(ops.NumericError):
            ops.modet_fwd(Qd, Kd, Bbad, dims, cfg, layout=MDG_QK_PLANAR)
    with torch.cuda.stream(streams[1]):
        d1, Q1, K1, B1, SF1 = cases[1]
        SF, _ = ops.modet_fwd(Q1, K1, B1, d1, cfg, layout=MDG_QK_PLANAR)
    torch.cuda.synchronize()
    assert rel_close(host(SF), SF1, FLOW_ATOL, FLOW_RTOL)


@pytest.mark.parametrize("variant", ["fused1", "fused2"])
@pytest.mark.parametrize("dims,S,hd", [((33, 17, 9), 1, 6), ((65, 3, 31), 2, 6), ((20, 24, 28), 4, 6),
                                       ((10, 12, 14), 2, 3), ((32, 16, 13), 1, 5)])
def test_single_pass_backward_variants(cuda, oracle, variant, dims, S, hd):
    """The single-pass ModeT backward kernels (MDG_MODET_BWD=fused1 / fused2:
    one logit evaluation per (source, window slot), the tile's source ring
    recomputed in-CTA, no atomics) against the oracle, in subprocesses since
    the variant is fixed at first use."""
    import subprocess
    import sys

    code = f"""
import sys, numpy as np, torch
sys.path[:0] = {[os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)), os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle")]!r}
import pyoracle
from _util import f32, random_qk
from test_gpu_modet import oracle_modet, run_fused, grad_ok, rel_close
from paper_2403_16526_b200._capi import MDG_QK_PLANAR
dims, S, hd = {dims!r}, {S}, {hd}
n = dims[0] * dims[1] * dims[2]
seed = sum(dims) * 5 + S + hd
Q = random_qk(dims, S * hd, seed); K = random_qk(dims, S * hd, seed + 1)
B = f32(pyoracle.Rng(seed + 2).normal(S * 27).reshape(S, 27))
gSF = f32(pyoracle.Rng(seed + 3).normal(3 * S * n).reshape(3 * S, dims[2], dims[1], dims[0]))
W0, SF0, gQ0, gK0, gB0 = oracle_modet(pyoracle.mdo(), Q, K, B, dims, S, hd, gSF)
for acc in (False, True):
    W, SF, LSE, gQ, gK, gB = run_fused(Q, K, B, dims, S, hd, gSF, MDG_QK_PLANAR, acc)
    assert grad_ok(gQ, gQ0) and grad_ok(gK, gK0), acc
    assert grad_ok(gB, gB0, 1e-4 if not acc else 1e-3), acc
print("ok")
"""
    env = dict(os.environ, MDG_MODET_BWD=variant)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
