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
    def __init__(self):
        self.store = {}

    def put(self, name, rank, x):
        self.store[(name, rank)] = x

    def __call__(self, name, x, sl, fill):
        self.store[(name, sl.rank)] = x
        C = x.shape[0]
        lo = torch.full((C, sl.w, sl.h), fill, device=x.device)
        hi = torch.full((C, sl.w, sl.h), fill, device=x.device)
        if sl.rank > 0:
            lo = self.store[(name, sl.rank - 1)][:, -1].clone()
        if sl.rank < sl.world - 1:
            hi = self.store[(name, sl.rank + 1)][:, 0].clone()
        return lo, hi


@pytest.mark.parametrize("world,dims,S,hd", [(2, (20, 12, 16), 1, 6), (3, (33, 9, 10), 2, 4),
                                              (4, (16, 16, 8), 1, 6)])
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

    ex = SimExchange()
    slabs = [slabmod.Slab(h, w, l, world, rk) for rk in range(world)]
    mods = [slabmod.SlabModeT(sl, S, hd, exchange=ex, all_reduce=lambda t: None) for sl in slabs]
    for sl in slabs:
        ex.put("K", sl.rank, sl.local(K))
    sfs = [m.forward(sl.local(Q), sl.local(K), B) for m, sl in zip(mods, slabs)]
    for m, sl in zip(mods, slabs):  # what each rank publishes before its backward
        _, _, _, sf, saved, _ = m._saved
        for name, t in (("Q", sl.local(Q)), ("SF", sf), ("saved", saved), ("gSF", sl.local(gSF))):
            ex.put(name, sl.rank, t)
    outs = [m.backward(sl.local(gSF)) for m, sl in zip(mods, slabs)]
    torch.cuda.synchronize()
    full = lambda t: t.reshape(t.shape[0], l, w, h).cpu().numpy()  # noqa: E731
    cat = lambda ts: np.concatenate([t.cpu().numpy() for t in ts], axis=1)  # noqa: E731
    assert np.array_equal(cat(sfs), full(SF))
    assert np.array_equal(cat([o[0] for o in outs]), full(gQ))
    assert np.array_equal(cat([o[1] for o in outs]), full(gK))
    gB_sum = sum(o[2] for o in outs)  # the all-reduce, done by hand here
    assert np.allclose(gB_sum.cpu().numpy(), gB.cpu().numpy(), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("world,dims,C,zreach", [(2, (20, 12, 16), 8, 2.5), (4, (16, 9, 12), 3, 4.2)])
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

    def exchange(name, x, sl, R_):
        lo, hi = max(0, sl.z0 - R_), min(l, sl.z1 + R_)
        return vol[:, lo:hi].clone()  # what the owners would send

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
