"""Depth-slab ModeT with the libmdg backend on one GPU: the ranks run one
after another in this process and a simulated exchange hands each rank its
neighbours' face planes (the multi-process exchange itself is covered over
gloo in tests/test_slab.py).  The stitched slab results must equal the
full-volume fused operator: SF, dQ, dK bit for bit (same per-voxel term
order), dB to fp32 reduction tolerance."""
import numpy as np
import pytest
import torch

from _util import f32
from paper_2403_16526_b200 import ops, slab as slabmod

pytestmark = pytest.mark.gpu


class SimExchange:
    """The neighbours' face planes, taken from the whole-volume tensors each
    rank's exchange would deliver (tag -> the packed global tensors)."""

    def __init__(self, tensors):
        self.t = tensors

    def start(self, tag, send_lo, send_hi, sl):
        g = torch.cat(self.t[tag])  # {sum C, l, w, h}
        lo = g[:, sl.z0 - 1].contiguous() if sl.rank > 0 else None
        hi = g[:, sl.z1].contiguous() if sl.rank < sl.world - 1 else None
        assert send_lo.shape == g[:, 0].shape

        class P:
            def wait(self):
                return lo, hi
        return P()


def _random_modet_cases(seed, count):
    r = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        world = int(r.integers(2, 5))
        out.append((world, (int(r.integers(2, 40)), int(r.integers(1, 20)),
                            int(r.integers(world, 4 * world + 4))),
                    int(r.choice([1, 2, 3])), int(r.choice([1, 2, 3, 4, 5, 6, 8]))))
    return out


@pytest.mark.parametrize("world,dims,S,hd", [(2, (20, 12, 16), 1, 6), (3, (33, 9, 10), 2, 4),
                                              (4, (16, 16, 8), 1, 6)] + _random_modet_cases(43, 8))
def test_slab_modet_cuda_matches_full_volume(cuda, world, dims, S, hd):
    h, w, l = dims
    r = np.random.default_rng(5)
    Q = torch.from_numpy(f32(r.standard_normal((S * hd, l, w, h)))).cuda()
    K = torch.from_numpy(f32(r.standard_normal((S * hd, l, w, h)))).cuda()
    B = torch.from_numpy(f32(r.uniform(-0.5, 0.5, (S, 27)))).cuda()
    gSF = torch.from_numpy(f32(r.uniform(-1, 1, (3 * S, l, w, h)))).cuda()
    cfg = ops.AttentionConfig(S, hd, 3)
    SF, LSE = ops.modet_fwd(Q, K, B, dims, cfg, layout=ops.MDG_QK_PLANAR)
    gQ, gK, gB = ops.modet_bwd(Q, K, B, SF, LSE, gSF, dims, cfg, layout=ops.MDG_QK_PLANAR)

    v = lambda t: t.reshape(t.shape[0], l, w, h)  # noqa: E731
    ex = SimExchange({"QK": [v(Q), v(K)], "SF": [v(SF), v(LSE), v(gSF)]})
    slabs = [slabmod.Slab(h, w, l, world, rk) for rk in range(world)]
    mods = [slabmod.SlabModeT(sl, S, hd, exchange=ex, all_reduce=lambda t: None) for sl in slabs]
    sfs = [m.forward(sl.local(Q), sl.local(K), B) for m, sl in zip(mods, slabs)]
    outs = [m.backward(sl.local(gSF)) for m, sl in zip(mods, slabs)]
    torch.cuda.synchronize()
    full = lambda t: t.reshape(t.shape[0], l, w, h).cpu().numpy()  # noqa: E731
    cat = lambda ts: np.concatenate([t.cpu().numpy() for t in ts], axis=1)  # noqa: E731
    assert np.array_equal(cat(sfs), full(SF))
    assert np.array_equal(cat([o[0] for o in outs]), full(gQ))
    assert np.array_equal(cat([o[1] for o in outs]), full(gK))
    gB_sum = sum(o[2] for o in outs)  # the all-reduce, done by hand here
    assert np.allclose(gB_sum.cpu().numpy(), gB.cpu().numpy(), rtol=1e-5, atol=1e-5)


def _random_slab_cases(seed, count):
    r = np.random.default_rng(seed)
    cases = []
    for _ in range(count):
        world = int(r.integers(2, 5))
        l = int(r.integers(world, 3 * world + 6))
        cases.append((world, (int(r.integers(2, 23)), int(r.integers(1, 13)), l),
                      int(r.choice([1, 2, 3, 4, 5, 8, 16])), float(r.uniform(0.2, 5.0))))
    return cases


@pytest.mark.parametrize("world,dims,C,zreach", [(2, (20, 12, 16), 8, 2.5), (4, (16, 9, 12), 3, 4.2)]
                         + _random_slab_cases(41, 10))
def test_slab_warp_cuda_matches_full_volume(cuda, world, dims, C, zreach):
    """SlabWarp with the libmdg range kernels, ranks run in turn with a
    simulated plane exchange / reduction: out and gfield equal the
    whole-volume warp bit for bit, gin to atomic-order tolerance."""
    h, w, l = dims
    r = np.random.default_rng(9)
    vol = torch.from_numpy(f32(r.standard_normal((C, l, w, h)))).cuda()
    fld = torch.from_numpy(f32(np.stack([r.uniform(-1.5, 1.5, (l, w, h)),
                                         r.uniform(-1.5, 1.5, (l, w, h)),
                                         r.uniform(-zreach, zreach, (l, w, h))]))).cuda()
    gout = torch.from_numpy(f32(r.standard_normal((C, l, w, h)))).cuda()
    out = ops.warp(vol, fld)
    gin, gfield = ops.warp_bwd(vol, fld, gout)

    slabs = [slabmod.Slab(h, w, l, world, rk) for rk in range(world)]
    R = max(slabmod.warp_reach(sl.local(fld), l) for sl in slabs)

    def exchange(name, x, sl, R_, out):
        lo, hi = max(0, sl.z0 - R_), min(l, sl.z1 + R_)
        out.copy_(vol[:, lo:hi])  # what the owners would send
        return out

    contribs = {}

    def reduce(name, c, sl, R_):
        acc = torch.zeros(c.shape[0], sl.depth, w, h, device=c.device)
        for q in slabs:  # rank order, as reduce_planes
            cq = contribs[q.rank]
            qlo = max(0, q.z0 - R_)
            a, b = max(sl.z0, qlo), min(sl.z1, qlo + cq.shape[1])
            if a < b:
                acc[:, a - sl.z0:b - sl.z0] += cq[:, a - qlo:b - qlo]
        return acc

    mods = [slabmod.SlabWarp(sl, exchange=exchange, reduce=reduce, all_reduce_max=lambda v: R)
            for sl in slabs]
    outs = [m.forward(sl.local(vol), sl.local(fld)) for m, sl in zip(mods, slabs)]
    loc = [m.backward_local(sl.local(gout)) for m, sl in zip(mods, slabs)]
    for sl, (c, _) in zip(slabs, loc):
        contribs[sl.rank] = c
    gins = [reduce("gin", loc[i][0], sl, R) for i, sl in enumerate(slabs)]
    torch.cuda.synchronize()
    cat = lambda ts: np.concatenate([t.cpu().numpy() for t in ts], axis=1)  # noqa: E731
    full = lambda t: t.reshape(t.shape[0], l, w, h).cpu().numpy()  # noqa: E731
    assert R > 1 and np.array_equal(cat(outs), full(out))
    assert np.array_equal(cat([g for _, g in loc]), full(gfield))
    assert np.allclose(cat(gins), full(gin), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("C", [1, 3, 5, 8, 16])
def test_warp_slab_abi_matches_range(cuda, C):
    """mdg_warp_fwd_slab / _bwd_slab on window-sized buffers equal the range
    kernels on full-size buffers (out, gfield bit for bit; gin to atomic
    order), and a field that leaves the window is refused, not followed."""
    h, w, l = 20, 12, 16
    r = np.random.default_rng(31 + C)
    vol = torch.from_numpy(f32(r.standard_normal((C, l, w, h)))).cuda()
    fld = torch.from_numpy(f32(np.stack([r.uniform(-1.5, 1.5, (l, w, h)),
                                         r.uniform(-1.5, 1.5, (l, w, h)),
                                         r.uniform(-2.5, 2.5, (l, w, h))]))).cuda()
    gout = torch.from_numpy(f32(r.standard_normal((C, l, w, h)))).cuda()
    L, P = ops._capi.lib(), ops._ptr
    d = ops.dims3((h, w, l))
    hw = h * w
    z0, z1, zi0, zi1 = 5, 11, 1, 15  # reach ceil(2.5) + 1 = 4 planes
    out_full = torch.zeros_like(vol)
    gin_full = torch.zeros_like(vol)
    gf_full = torch.zeros_like(fld)
    ops._check(L.mdg_warp_fwd_range(P(vol), C, d, P(fld), P(out_full), z0 * hw, z1 * hw,
                                    ops._stream()))
    ops._check(L.mdg_warp_bwd_range(P(vol), C, d, P(fld), P(gout), P(gin_full), P(gf_full),
                                    z0 * hw, z1 * hw, ops._stream()))
    win = vol[:, zi0:zi1].contiguous()
    f_s, go_s = fld[:, z0:z1].contiguous(), gout[:, z0:z1].contiguous()
    out_s = torch.zeros(C, z1 - z0, w, h, device="cuda")
    gin_s = torch.zeros(C, zi1 - zi0, w, h, device="cuda")
    gf_s = torch.zeros(3, z1 - z0, w, h, device="cuda")
    ops._check(L.mdg_warp_fwd_slab(P(win), C, d, zi0, zi1, P(f_s), P(out_s), z0, z1,
                                   ops._stream()))
    ops._check(L.mdg_warp_bwd_slab(P(win), C, d, zi0, zi1, P(f_s), P(go_s), P(gin_s), P(gf_s),
                                   z0, z1, ops._stream()))
    torch.cuda.synchronize()
    assert torch.equal(out_s, out_full[:, z0:z1])
    assert torch.equal(gf_s, gf_full[:, z0:z1])
    assert not gin_full[:, :zi0].any() and not gin_full[:, zi1:].any()
    assert torch.allclose(gin_s, gin_full[:, zi0:zi1], rtol=1e-5, atol=1e-5)
    # a window short of the reach: refused (EINVAL; the out-of-window voxels
    # touch nothing — compute-sanitizer clean)
    small = vol[:, 4:12].contiguous()
    with pytest.raises(ops.InvalidInput, match="outside the input window"):
        ops._check(L.mdg_warp_bwd_slab(P(small), C, d, 4, 12, P(f_s), P(go_s),
                                       P(gin_s[:, :8].contiguous()), P(gf_s), z0, z1,
                                       ops._stream()))
    with pytest.raises(ops.InvalidInput, match="outside the input window"):
        ops._check(L.mdg_warp_fwd_slab(P(small), C, d, 4, 12, P(f_s), P(out_s),
                                       z0, z1, ops._stream()))
    with pytest.raises(ops.InvalidInput, match="must cover"):
        ops._check(L.mdg_warp_fwd_slab(P(win), C, d, 6, 15, P(f_s), P(out_s), z0, z1,
                                       ops._stream()))
