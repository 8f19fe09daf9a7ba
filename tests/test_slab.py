"""Depth-slab decomposition of the ModeT operator (paper_2403_16526_b200/slab.py).

CPU: world_size 2 and 3 over gloo, each rank running the SAME decomposition
with the CPU oracle as compute backend; the stitched slab results must equal
the full-volume oracle bit for bit (SF, gQ, gK: identical per-element term
order) and gB to fp32 reduction tolerance (summed across ranks).
GPU (tests/test_gpu_slab.py) drives the libmdg backend through the same class.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from _util import f32
from paper_2403_16526_b200 import slab as slabmod


def test_split_balanced():
    assert slabmod.split(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert slabmod.split(4, 4) == [(0, 1), (1, 2), (2, 3), (3, 4)]
    assert slabmod.split(7, 1) == [(0, 7)]
    with pytest.raises(ValueError):
        slabmod.split(2, 3)


class OracleModeT:
    """Test backend: the CPU oracle (mdo) on the extended slab.  Saved
    statistics are the softmax rows W (planar {S*27, n}); halo rows at the
    global boundary are 0 (phantom sources carry no weight)."""

    saved_fill = 0.0

    def __init__(self, S, hd):
        import pyoracle

        self.m = pyoracle.mdo()
        self.S, self.hd = S, hd

    def _pm(self, x, n):  # planar {C, ...} -> position-major {n, C}
        return f32(x.reshape(x.shape[0], n).T.numpy())

    def forward(self, Qx, Kx, B, dims):
        h, w, l = dims
        n = h * w * l
        W, bad = self.m.na_fwd(self._pm(Qx, n), self._pm(Kx, n), f32(B.numpy()), dims, self.S,
                               self.hd)
        assert bad is None
        SF = torch.from_numpy(self.m.subfields_fwd(W, dims, self.S))
        Wp = torch.from_numpy(f32(W.transpose(0, 2, 1).reshape(self.S * 27, l, w, h)))
        return SF, Wp

    def _bwd(self, Qx, Kx, savedx, gSF, dims):
        h, w, l = dims
        n = h * w * l
        W = f32(savedx.numpy().reshape(self.S, 27, n).transpose(0, 2, 1))
        gW = self.m.subfields_bwd(f32(gSF.numpy()), dims, self.S)
        gQ, gK, gB = self.m.na_bwd(self._pm(Qx, n), self._pm(Kx, n), W, gW, dims, self.S, self.hd)
        pl = lambda a: torch.from_numpy(f32(a.T.reshape(-1, l, w, h)))  # noqa: E731
        return pl(gQ), pl(gK), torch.from_numpy(gB)

    def backward_queries(self, Qx, Kx, B, SFx, savedx, gSF_rows, dims, gB):
        gQ, _, gb = self._bwd(Qx, Kx, savedx, gSF_rows, dims)
        gB += gb
        return gQ

    def backward_keys(self, Qx, Kx, B, SFx, savedx, gSFx, dims):
        return self._bwd(Qx, Kx, savedx, gSFx, dims)[1]


def _case(dims, S, hd, seed):
    h, w, l = dims
    r = np.random.default_rng(seed)
    Q = f32(r.standard_normal((S * hd, l, w, h)))
    K = f32(r.standard_normal((S * hd, l, w, h)))
    B = f32(r.uniform(-0.5, 0.5, (S, 27)))
    gSF = f32(r.uniform(-1, 1, (3 * S, l, w, h)))
    return Q, K, B, gSF


def _worker(rank, world, port, dims, S, hd, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Q, K, B, gSF = (torch.from_numpy(a) for a in _case(dims, S, hd, seed=11))
        sl = slabmod.Slab(*dims, world=world, rank=rank)
        op = slabmod.SlabModeT(sl, S, hd, backend=OracleModeT(S, hd))
        SF = op.forward(sl.local(Q), sl.local(K), B)
        gQ, gK, gB = op.backward(sl.local(gSF))
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), SF=SF.numpy(), gQ=gQ.numpy(),
                 gK=gK.numpy(), gB=gB.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,dims,S,hd", [(2, (6, 5, 7), 1, 6), (3, (5, 4, 7), 2, 3)])
def test_slab_modet_over_gloo_matches_full_volume(oracle, tmp_path, world, dims, S, hd):
    mp.start_processes(_worker, args=(world, _free_port(), dims, S, hd, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    Q, K, B, gSF = _case(dims, S, hd, seed=11)
    h, w, l = dims
    n = h * w * l
    be = OracleModeT(S, hd)
    SF, Wp = be.forward(torch.from_numpy(Q), torch.from_numpy(K), torch.from_numpy(B), dims)
    gB = torch.zeros(S, 27)
    gQ = be.backward_queries(torch.from_numpy(Q), torch.from_numpy(K), None, None, Wp,
                             torch.from_numpy(gSF), dims, gB)
    gK = be.backward_keys(torch.from_numpy(Q), torch.from_numpy(K), None, None, Wp,
                          torch.from_numpy(gSF), dims)
    parts = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]
    cat = lambda k: np.concatenate([p[k] for p in parts], axis=1)  # noqa: E731
    assert np.array_equal(cat("SF"), SF.numpy())
    assert np.array_equal(cat("gQ"), gQ.numpy())
    assert np.array_equal(cat("gK"), gK.numpy())
    for p in parts:  # all-reduced: identical on every rank
        assert np.array_equal(p["gB"], parts[0]["gB"])
    assert np.allclose(parts[0]["gB"], gB.numpy(), rtol=1e-5, atol=1e-6)


# ------------------------------------------------------------ slab warp
class OracleWarp:
    """Test backend for SlabWarp: the CPU oracle's whole-volume warp, used
    over the rank's voxel range only."""

    def __init__(self):
        import pyoracle

        self.m = pyoracle.mdo()

    def _full(self, x, dims, z0):
        h, w, l = dims
        f = torch.zeros(x.shape[0], l, w, h, dtype=x.dtype)
        f[:, z0:z0 + x.shape[1]] = x
        return f

    def fwd_slab(self, win, field, out, dims, zi0, zi1, z0, z1):
        o = self.m.warp_fwd(f32(self._full(win, dims, zi0).numpy()),
                            f32(self._full(field, dims, z0).numpy()))
        out.copy_(torch.from_numpy(o[:, z0:z1]))

    def bwd_slab(self, win, field, gout, gin_win, gfield, dims, zi0, zi1, z0, z1):
        # gout zero outside the slab: only the slab's voxels scatter
        gi, gf = self.m.warp_bwd(f32(self._full(win, dims, zi0).numpy()),
                                 f32(self._full(field, dims, z0).numpy()),
                                 f32(self._full(gout, dims, z0).numpy()))
        gin_win += torch.from_numpy(gi[:, zi0:zi1])
        gfield.copy_(torch.from_numpy(gf[:, z0:z1]))


def _warp_case(dims, C, seed, zreach):
    h, w, l = dims
    r = np.random.default_rng(seed)
    vol = f32(r.standard_normal((C, l, w, h)))
    fld = f32(np.stack([r.uniform(-1.5, 1.5, (l, w, h)), r.uniform(-1.5, 1.5, (l, w, h)),
                        r.uniform(-zreach, zreach, (l, w, h))]))
    gout = f32(r.standard_normal((C, l, w, h)))
    return vol, fld, gout


def _warp_worker(rank, world, port, dims, C, zreach, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vol, fld, gout = (torch.from_numpy(a) for a in _warp_case(dims, C, 21, zreach))
        sl = slabmod.Slab(*dims, world=world, rank=rank)
        op = slabmod.SlabWarp(sl, backend=OracleWarp())
        out = op.forward(sl.local(vol), sl.local(fld))
        gin, gfield = op.backward(sl.local(gout))
        np.savez(os.path.join(out_dir, f"w{rank}.npz"), out=out.numpy(), gin=gin.numpy(),
                 gfield=gfield.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,C,zreach", [(2, (6, 5, 7), 3, 1.7), (3, (5, 4, 9), 2, 3.6)])
def test_slab_warp_over_gloo_matches_full_volume(oracle, tmp_path, world, dims, C, zreach):
    """z reach all-reduced, planes gathered from (possibly several) owning
    ranks, the scattered input gradient returned to its owners: out and
    gfield bit for bit, gin to summation-order tolerance."""
    mp.start_processes(_warp_worker, args=(world, _free_port(), dims, C, zreach, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    vol, fld, gout = _warp_case(dims, C, 21, zreach)
    be = OracleWarp()
    out = be.m.warp_fwd(vol, fld)
    gin, gfield = be.m.warp_bwd(vol, fld, gout)
    parts = [dict(np.load(tmp_path / f"w{r}.npz")) for r in range(world)]
    cat = lambda k: np.concatenate([p[k] for p in parts], axis=1)  # noqa: E731
    assert np.array_equal(cat("out"), out)
    assert np.array_equal(cat("gfield"), gfield)
    assert np.allclose(cat("gin"), gin, rtol=1e-5, atol=1e-5)


def test_warp_reach():
    f = torch.zeros(3, 4, 3, 3)
    assert slabmod.warp_reach(f, 10) == 1
    f[2, 1, 1, 1] = -2.3
    assert slabmod.warp_reach(f, 10) == 4
    f[2, 0, 0, 0] = float("nan")
    assert slabmod.warp_reach(f, 10) == 10
