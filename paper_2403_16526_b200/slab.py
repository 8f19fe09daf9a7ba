"""Depth-slab decomposition of the ModeT operator across ranks (SURVEY §8e,
"Depth-slab (cfg3, cfg4)").

The volume is split along z — the slowest, contiguous axis (common.hpp:56-59)
— into one slab per rank.  The operator's 3x3x3 window reaches one plane
across each slab face, so every rank works on its slab extended by one halo
plane per side:

* forward: the K halo planes come from the neighbours (point-to-point
  send/recv, NCCL over NVLink on GPUs); Q halo planes are zero (their outputs
  are discarded).  Zero K at the GLOBAL boundary is exactly the reference's
  out-of-bounds rule (attention.hpp:77-81: the term is omitted, logit = bias;
  q . 0 = 0 gives the same logit).
* backward: halos of Q, K, the saved softmax statistics (LSE), SF and gSF.
  The query-side pass (dQ, dB) runs with the halo planes' gSF zeroed, so halo
  queries contribute nothing (they belong to the neighbour); the key-side pass
  (dK, a gather over sources r = q - off(o)) runs with the true halo gSF, so
  keys on the slab face collect the contributions of sources in the
  neighbour's planes.  At the global boundary the halo is empty: LSE = +inf
  makes those phantom sources weigh exactly 0.
* dB (the relative-position bias gradient) is the only quantity summed over
  ranks: one all-reduce of S*27 floats.

The compute backend is pluggable for testing (tests/test_slab.py drives the
same decomposition with the CPU oracle over gloo); the product backend is
:class:`CudaModeT` — libmdg's fused kernels, with no fallback.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def split(l: int, world: int):
    """Balanced z ranges [(z0, z1)] for `world` ranks (earlier ranks get the
    remainder).  Every rank needs at least one plane."""
    if world < 1 or l < world:
        raise ValueError(f"slab: cannot split {l} planes over {world} ranks")
    base, rem = divmod(l, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((z, z + n))
        z += n
    return out


@dataclass
class Slab:
    """This rank's piece of a {*, l, w, h} volume."""

    h: int
    w: int
    l: int  # global depth
    world: int
    rank: int

    def __post_init__(self):
        self.z0, self.z1 = split(self.l, self.world)[self.rank]

    @property
    def depth(self) -> int:
        return self.z1 - self.z0

    @property
    def dims(self):
        """local dims (h, w, depth)"""
        return (self.h, self.w, self.depth)

    @property
    def ext_dims(self):
        """dims of the slab plus one halo plane per side"""
        return (self.h, self.w, self.depth + 2)

    def local(self, full: torch.Tensor) -> torch.Tensor:
        """This rank's planes of a planar {C, l, w, h} (or {C, n}) tensor."""
        C = full.shape[0]
        v = full.reshape(C, self.l, self.w, self.h)
        return v[:, self.z0:self.z1].contiguous()


def exchange_halo(x: torch.Tensor, slab: Slab, fill: float = 0.0, group=None):
    """x: local planes {C, depth, w, h}.  Returns the neighbours' adjacent
    planes (lo = plane z0-1, hi = plane z1), each {C, w, h}; `fill` where the
    neighbour does not exist (global boundary)."""
    C = x.shape[0]
    lo = torch.full((C, slab.w, slab.h), fill, dtype=x.dtype, device=x.device)
    hi = torch.full((C, slab.w, slab.h), fill, dtype=x.dtype, device=x.device)
    if slab.world == 1:
        return lo, hi
    first = x[:, 0].contiguous()
    last = x[:, -1].contiguous()
    ops = []
    if slab.rank > 0:
        ops.append(dist.P2POp(dist.isend, first, slab.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, lo, slab.rank - 1, group))
    if slab.rank < slab.world - 1:
        ops.append(dist.P2POp(dist.isend, last, slab.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, hi, slab.rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    return lo, hi


def extend(x: torch.Tensor, lo: torch.Tensor, hi: torch.Tensor) -> torch.Tensor:
    """[lo, x, hi] along z: {C, depth+2, w, h}."""
    return torch.cat([lo.unsqueeze(1), x, hi.unsqueeze(1)], dim=1).contiguous()


def interior(x_ext: torch.Tensor) -> torch.Tensor:
    return x_ext[:, 1:-1].contiguous()


class CudaModeT:
    """Product backend: libmdg's fused ModeT kernels on the extended slab
    (planar Q/K, saved statistics = LSE {S, n})."""

    saved_fill = float("inf")  # phantom sources beyond the global boundary

    def __init__(self, heads: int, head_dim: int):
        from . import ops

        self.ops = ops
        self.cfg = ops.AttentionConfig(heads, head_dim, 3)

    def forward(self, Q_ext, K_ext, B, dims):
        SF, LSE = self.ops.modet_fwd(Q_ext, K_ext, B, dims, self.cfg,
                                     layout=self.ops.MDG_QK_PLANAR, check=False)
        h, w, l = dims
        return SF.view(-1, l, w, h), LSE.view(-1, l, w, h)

    def check(self, dims):
        self.ops.check_numeric(dims)

    def backward_queries(self, Q_ext, K_ext, B, SF_ext, saved_ext, gSF_rows, dims, gB):
        gQ = torch.empty_like(Q_ext)
        self._bwd(Q_ext, K_ext, B, SF_ext, saved_ext, gSF_rows, dims, gQ, None, gB)
        return gQ

    def backward_keys(self, Q_ext, K_ext, B, SF_ext, saved_ext, gSF_ext, dims):
        gK = torch.empty_like(K_ext)
        self._bwd(Q_ext, K_ext, B, SF_ext, saved_ext, gSF_ext, dims, None, gK, None)
        return gK

    def _bwd(self, Q, K, B, SF, LSE, gSF, dims, gQ, gK, gB):
        o = self.ops
        P = o._ptr
        L = o._capi.lib()
        o._check(L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(gSF), o.dims3(dims),
                                 self.cfg.heads, self.cfg.head_dim, 3, o.MDG_QK_PLANAR,
                                 P(gQ), P(gK), P(gB), 0, o._stream()))


class SlabModeT:
    """ModeT forward/backward on this rank's z-slab with halo exchange.

    Tensors are planar and local: Q, K {S*d, depth, w, h}; B {S, 27} (same on
    every rank); outputs SF {3S, depth, w, h}; the backward returns local
    gQ, gK and the all-reduced gB."""

    def __init__(self, slab: Slab, heads: int, head_dim: int, backend=None, group=None,
                 exchange=None, all_reduce=None):
        self.slab, self.S, self.hd = slab, heads, head_dim
        self.be = backend if backend is not None else CudaModeT(heads, head_dim)
        self.group = group
        # exchange(name, x, slab, fill) -> (lo, hi); the default is the
        # point-to-point exchange over the process group
        self.exchange = exchange or (lambda name, x, sl, fill: exchange_halo(x, sl, fill, group))
        self.all_reduce = all_reduce or (
            lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group))
        self._saved = None

    def _ext(self, name, x, fill=0.0):
        lo, hi = self.exchange(name, x, self.slab, fill)
        return extend(x, lo, hi)

    def forward(self, Q, K, B):
        s = self.slab
        if s.world == 1 and isinstance(self.be, CudaModeT):
            # one slab = the whole volume: the fused operator directly
            SF, LSE = self.be.forward(Q, K, B, s.dims)
            self.be.check(s.dims)
            self._saved = (Q, K, B, SF, LSE, True)
            return SF
        Kx = self._ext("K", K)
        zero = torch.zeros(Q.shape[0], s.w, s.h, dtype=Q.dtype, device=Q.device)
        Qx = extend(Q, zero, zero)  # halo queries are the neighbours' work
        SFx, saved_x = self.be.forward(Qx, Kx, B, s.ext_dims)
        if hasattr(self.be, "check"):
            try:
                self.be.check(s.ext_dims)
            except Exception as e:  # report the global position
                pos = getattr(e, "position", None)
                if pos is not None and pos[2] >= 0:
                    e.position = (pos[0], pos[1], pos[2] - 1 + s.z0, pos[3])
                raise
        SF, saved = interior(SFx), interior(saved_x)
        self._saved = (Q, K, B, SF, saved, False)
        return SF

    def backward(self, gSF):
        if self._saved is None:
            raise RuntimeError("slab: backward without forward")
        Q, K, B, SF, saved, whole = self._saved
        s = self.slab
        if whole:
            gB = torch.zeros_like(B)
            gQ = torch.empty_like(Q)
            gK = torch.empty_like(K)
            self.be._bwd(Q, K, B, SF, saved, gSF, s.dims, gQ, gK, gB)
            return gQ, gK, gB
        Qx, Kx = self._ext("Q", Q), self._ext("K", K)
        SFx, gSFx = self._ext("SF", SF), self._ext("gSF", gSF)
        savedx = self._ext("saved", saved, fill=self.be.saved_fill)
        zero = torch.zeros(gSF.shape[0], s.w, s.h, dtype=gSF.dtype, device=gSF.device)
        gSF_rows = extend(gSF, zero, zero)
        gB = torch.zeros_like(B)
        gQx = self.be.backward_queries(Qx, Kx, B, SFx, savedx, gSF_rows, s.ext_dims, gB)
        gKx = self.be.backward_keys(Qx, Kx, B, SFx, savedx, gSFx, s.ext_dims)
        if s.world > 1:
            self.all_reduce(gB)
        return interior(gQx), interior(gKx), gB


# ----------------------------------------------------------------- the warp
# The trilinear warp's reach is data-dependent: voxel p reads (and its
# backward scatters into) the z rows floor(z + phi_z) and +1, so a slab needs
# R = ceil(max |phi_z|) + 1 planes beyond each face ("Warp:
# ceil(max|phi_z|)+1 planes after an ncclAllReduce(max)").  R is all-reduced
# so every rank knows every other rank's range; planes then move point to
# point between the owning and the needing ranks (a halo may span several
# slabs when R exceeds a slab's depth).  Each rank runs the warp kernels over
# its own voxel range in GLOBAL coordinates (full-size buffers, global dims),
# so clamping and the boundary rules are the whole-volume ones: out and
# gfield are identical to the whole-volume call.  The scattered input
# gradient's contributions to other ranks' planes are sent back and summed by
# the owner in rank order.


def warp_reach(field_local: torch.Tensor, l: int) -> int:
    """ceil(max |phi_z|) + 1 over this rank's voxels (the whole depth if any
    z displacement is non-finite)."""
    fz = field_local[2]
    if fz.numel() == 0:
        return 1
    if not bool(torch.isfinite(fz).all()):
        return l
    return min(l, int(torch.ceil(fz.abs().max()).item()) + 1)


def _need(sl: Slab, z0: int, z1: int, R: int):
    return max(0, z0 - R), min(sl.l, z1 + R)


def _p2p(ops_list):
    if ops_list:
        for req in dist.batch_isend_irecv(ops_list):
            req.wait()


def exchange_planes(x: torch.Tensor, sl: Slab, R: int, group=None) -> torch.Tensor:
    """Global planes [z0-R, z1+R) (clipped) of a {C, depth, w, h} slab-local
    tensor, gathered from their owners."""
    ranges = split(sl.l, sl.world)
    lo, hi = _need(sl, sl.z0, sl.z1, R)
    C = x.shape[0]
    out = torch.empty(C, hi - lo, sl.w, sl.h, dtype=x.dtype, device=x.device)
    out[:, sl.z0 - lo:sl.z1 - lo] = x
    ops_list, keep = [], []
    for q, (a, b) in enumerate(ranges):
        if q == sl.rank:
            continue
        qlo, qhi = _need(sl, a, b, R)
        s0, s1 = max(sl.z0, qlo), min(sl.z1, qhi)  # mine, needed by q
        if s0 < s1:
            t = x[:, s0 - sl.z0:s1 - sl.z0].contiguous()
            keep.append(t)
            ops_list.append(dist.P2POp(dist.isend, t, q, group))
        r0, r1 = max(a, lo), min(b, hi)  # q's, needed by me
        if r0 < r1:
            t = torch.empty(C, r1 - r0, sl.w, sl.h, dtype=x.dtype, device=x.device)
            keep.append((t, r0))
            ops_list.append(dist.P2POp(dist.irecv, t, q, group))
    _p2p(ops_list)
    for item in keep:
        if isinstance(item, tuple):
            t, r0 = item
            out[:, r0 - lo:r0 - lo + t.shape[1]] = t
    return out


def reduce_planes(contrib: torch.Tensor, sl: Slab, R: int, group=None) -> torch.Tensor:
    """contrib: this rank's additions to the global planes [z0-R, z1+R)
    (clipped).  Returns this rank's planes summed over all ranks' additions,
    in rank order."""
    ranges = split(sl.l, sl.world)
    lo, hi = _need(sl, sl.z0, sl.z1, R)
    ops_list, recvd = [], {}
    for q, (a, b) in enumerate(ranges):
        if q == sl.rank:
            continue
        s0, s1 = max(a, lo), min(b, hi)  # my additions to q's planes
        if s0 < s1:
            ops_list.append(dist.P2POp(dist.isend, contrib[:, s0 - lo:s1 - lo].contiguous(), q,
                                       group))
        qlo, qhi = _need(sl, a, b, R)
        r0, r1 = max(sl.z0, qlo), min(sl.z1, qhi)  # q's additions to mine
        if r0 < r1:
            t = torch.empty(contrib.shape[0], r1 - r0, sl.w, sl.h, dtype=contrib.dtype,
                            device=contrib.device)
            recvd[q] = (t, r0)
            ops_list.append(dist.P2POp(dist.irecv, t, q, group))
    _p2p(ops_list)
    out = torch.zeros(contrib.shape[0], sl.depth, sl.w, sl.h, dtype=contrib.dtype,
                      device=contrib.device)
    for q in range(sl.world):  # fixed order
        if q == sl.rank:
            out += contrib[:, sl.z0 - lo:sl.z1 - lo]
        elif q in recvd:
            t, r0 = recvd[q]
            out[:, r0 - sl.z0:r0 - sl.z0 + t.shape[1]] += t
    return out


class CudaWarp:
    """Product backend: libmdg's warp kernels over a voxel range of full-size
    buffers (mdg_warp_fwd_range / mdg_warp_bwd_range)."""

    def fwd_range(self, vol, field, out, dims, pb, pe):
        from . import ops

        L = ops._capi.lib()
        P = ops._ptr
        ops._check(L.mdg_warp_fwd_range(P(vol), vol.shape[0], ops.dims3(dims), P(field), P(out),
                                        pb, pe, ops._stream()))

    def bwd_range(self, vol, field, gout, gin, gfield, dims, pb, pe):
        from . import ops

        L = ops._capi.lib()
        P = ops._ptr
        ops._check(L.mdg_warp_bwd_range(P(vol), vol.shape[0], ops.dims3(dims), P(field), P(gout),
                                        P(gin), P(gfield), pb, pe, ops._stream()))


class SlabWarp:
    """Trilinear warp forward/backward on this rank's z-slab.  in {C, depth,
    w, h}, field {3, depth, w, h} (this rank's voxels' displacements, global
    voxel units); forward returns the rank's warped planes, backward (of the
    last forward) the rank's gin and gfield (fresh, not accumulated)."""

    def __init__(self, slab: Slab, backend=None, group=None, exchange=None, reduce=None,
                 all_reduce_max=None):
        self.slab = slab
        self.be = backend if backend is not None else CudaWarp()
        self.group = group
        self.exchange = exchange or (lambda name, x, sl, R: exchange_planes(x, sl, R, group))
        self.reduce = reduce or (lambda name, c, sl, R: reduce_planes(c, sl, R, group))

        def _max(v):
            t = torch.tensor([v], dtype=torch.int64)
            if slab.world > 1:
                if dist.get_backend(group) == "nccl":
                    t = t.cuda()
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            return int(t.item())

        self.all_reduce_max = all_reduce_max or _max
        self._saved = None
        self._bufs = {}

    def _full(self, name, C, ref):
        """persistent full-size buffer: the kernels only read the planes each
        call refreshes (the reach window, this rank's voxels), so stale planes
        elsewhere are never touched"""
        s = self.slab
        key = (name, C, ref.dtype, ref.device)
        b = self._bufs.get(key)
        if b is None:
            b = torch.zeros(C, s.l, s.w, s.h, dtype=ref.dtype, device=ref.device)
            self._bufs[key] = b
        return b

    def forward(self, vol, field):
        s = self.slab
        if s.world == 1 and isinstance(self.be, CudaWarp):
            # one slab = the whole volume: the whole-volume kernels directly
            out = torch.empty_like(vol)
            self.be.fwd_range(vol, field, out, (s.h, s.w, s.l), 0, s.h * s.w * s.l)
            self._saved = (vol, field, None)
            return out
        R = self.all_reduce_max(warp_reach(field, s.l))
        lo, hi = _need(s, s.z0, s.z1, R)
        C = vol.shape[0]
        vol_full, field_full = self._full("in", C, vol), self._full("field", 3, field)
        vol_full[:, lo:hi] = self.exchange("in", vol, s, R)
        field_full[:, s.z0:s.z1] = field
        out_full = self._full("out", C, vol)
        hw = s.h * s.w
        dims = (s.h, s.w, s.l)
        self.be.fwd_range(vol_full, field_full, out_full, dims, s.z0 * hw, s.z1 * hw)
        self._saved = (vol_full, field_full, R)
        return out_full[:, s.z0:s.z1].contiguous()

    def backward_local(self, gout):
        """(this rank's gin additions to planes [z0-R, z1+R), its gfield)"""
        if self._saved is None:
            raise RuntimeError("slab: backward without forward")
        vol_full, field_full, R = self._saved
        s = self.slab
        hw = s.h * s.w
        if R is None:  # world == 1: whole-volume kernels on the caller's tensors
            gin, gfield = torch.zeros_like(vol_full), torch.zeros_like(field_full)
            self.be.bwd_range(vol_full, field_full, gout, gin, gfield, (s.h, s.w, s.l), 0,
                              s.l * hw)
            return gin, gfield
        C = vol_full.shape[0]
        lo, hi = _need(s, s.z0, s.z1, R)
        gout_full = self._full("gout", C, gout)
        gin_full, gfield_full = self._full("gin", C, gout), self._full("gfield", 3, gout)
        gout_full[:, s.z0:s.z1] = gout
        gin_full[:, lo:hi].zero_()  # the scatter's reach
        gfield_full[:, s.z0:s.z1].zero_()
        self.be.bwd_range(vol_full, field_full, gout_full, gin_full, gfield_full,
                          (s.h, s.w, s.l), s.z0 * hw, s.z1 * hw)
        return gin_full[:, lo:hi].clone(), gfield_full[:, s.z0:s.z1].clone()

    def backward(self, gout):
        contrib, gfield = self.backward_local(gout)
        if self._saved[2] is None:  # world == 1: contrib is the whole gin
            return contrib, gfield
        gin = self.reduce("gin", contrib, self.slab, self._saved[2])
        return gin, gfield
