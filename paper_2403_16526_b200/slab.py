"""Depth-slab decomposition of the ModeT operator across ranks (SURVEY §8e,
"Depth-slab (cfg3, cfg4)").

The volume is split along z — the slowest, contiguous axis (common.hpp:56-59)
— into one slab per rank.  The operator's 3x3x3 window reaches one plane
across each slab face, so every rank works on its slab extended by one halo
plane per side:

* forward: the Q and K halo planes come from the neighbours (point-to-point
  send/recv, NCCL over NVLink on GPUs; the halo queries' outputs are
  discarded, their Q is kept for the backward).  Zero K at the GLOBAL
  boundary is exactly the reference's out-of-bounds rule (attention.hpp:77-81:
  the term is omitted, logit = bias; q . 0 = 0 gives the same logit).
* backward: halos of the saved softmax statistics (LSE), SF and gSF.
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


class HaloExchange:
    """Point-to-point exchange of face planes with the z neighbours.

    start(tag, send_lo, send_hi, slab) posts the sends of this rank's first
    (send_lo, to rank-1) and last (send_hi, to rank+1) planes and the
    receives of the neighbours' adjacent planes, and returns a handle whose
    wait() gives (recv_lo, recv_hi) — None where there is no neighbour (the
    global boundary).  With NCCL the transfers run on NCCL's stream, so work
    the caller launches between start() and wait() overlaps them; wait()
    only orders the caller's stream after them."""

    def __init__(self, group=None):
        self.group = group

    def start(self, tag, send_lo, send_hi, sl):
        recv_lo = torch.empty_like(send_lo) if sl.rank > 0 else None
        recv_hi = torch.empty_like(send_hi) if sl.rank < sl.world - 1 else None
        ops_ = []
        if recv_lo is not None:
            ops_.append(dist.P2POp(dist.isend, send_lo, sl.rank - 1, self.group))
            ops_.append(dist.P2POp(dist.irecv, recv_lo, sl.rank - 1, self.group))
        if recv_hi is not None:
            ops_.append(dist.P2POp(dist.isend, send_hi, sl.rank + 1, self.group))
            ops_.append(dist.P2POp(dist.irecv, recv_hi, sl.rank + 1, self.group))
        reqs = dist.batch_isend_irecv(ops_) if ops_ else []
        return _Pending(reqs, recv_lo, recv_hi, (send_lo, send_hi))


class _Pending:
    def __init__(self, reqs, lo, hi, keep):
        self.reqs, self.lo, self.hi, self._keep = reqs, lo, hi, keep

    def wait(self):
        for r in self.reqs:
            r.wait()
        self.reqs = []
        return self.lo, self.hi


def _faces(xs):
    """first and last interior planes of extended {C, D+2, w, h} tensors,
    packed over the channels: ({sum C, w, h}, {sum C, w, h})"""
    D = xs[0].shape[1] - 2
    return (torch.cat([x[:, 1] for x in xs]).contiguous(),
            torch.cat([x[:, D] for x in xs]).contiguous())


def _unpack(xs, recv, plane):
    """write the packed planes `recv` into plane `plane` of each tensor"""
    if recv is None:
        return
    c0 = 0
    for x in xs:
        c1 = c0 + x.shape[0]
        x[:, plane].copy_(recv[c0:c1])
        c0 = c1


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
    every rank); forward returns SF {3S, depth, w, h}; backward the local gQ,
    gK and the all-reduced gB.  Outputs are views of the extended
    {C, depth+2, w, h} working tensors (no interior copies).

    Memory and traffic: Q, K and gSF live in persistent extended buffers
    whose halo planes are written in place by the exchange.  A caller that
    writes its inputs into `input_views()` / `grad_view()` skips even the one
    copy into them.  The forward exchanges the Q and K faces (one packed
    message per neighbour); the backward's exchange of the SF, LSE and gSF
    faces runs on NCCL's stream while the query-side pass (dQ, dB) computes —
    that pass reads the halo rows with gSF = 0, so it needs none of them —
    and the key-side pass (dK) starts once they have landed."""

    def __init__(self, slab: Slab, heads: int, head_dim: int, backend=None, group=None,
                 exchange=None, all_reduce=None):
        self.slab, self.S, self.hd = slab, heads, head_dim
        self.be = backend if backend is not None else CudaModeT(heads, head_dim)
        self.group = group
        self.exchange = exchange or HaloExchange(group)
        self.all_reduce = all_reduce or (
            lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group))
        self._saved = None
        self._bufs = {}

    def _buf(self, name, C, like):
        """persistent extended buffer {C, depth+2, w, h}; halo planes zero
        until an exchange writes them"""
        s = self.slab
        key = (name, C, like.dtype, like.device)
        b = self._bufs.get(key)
        if b is None:
            b = torch.zeros(C, s.depth + 2, s.w, s.h, dtype=like.dtype, device=like.device)
            self._bufs[key] = b
        return b

    def input_views(self, like: torch.Tensor):
        """(Q, K) interior views of the extended input buffers: inputs written
        there are used in place"""
        C = self.S * self.hd
        return self._buf("Q", C, like)[:, 1:-1], self._buf("K", C, like)[:, 1:-1]

    def grad_view(self, like: torch.Tensor):
        """interior view of the extended gSF buffer (see input_views)"""
        return self._buf("gSF", 3 * self.S, like)[:, 1:-1]

    def _stage(self, name, x):
        b = self._buf(name, x.shape[0], x)
        v = b[:, 1:-1]
        if not (x.data_ptr() == v.data_ptr() and x.shape == v.shape and x.stride() == v.stride()):
            v.copy_(x.reshape(v.shape))
        return b

    def forward(self, Q, K, B):
        s = self.slab
        if s.world == 1 and isinstance(self.be, CudaModeT):
            # one slab = the whole volume: the fused operator directly
            SF, LSE = self.be.forward(Q, K, B, s.dims)
            self.be.check(s.dims)
            self._saved = (Q, K, B, SF, LSE, True)
            return SF
        Qx, Kx = self._stage("Q", Q), self._stage("K", K)
        lo, hi = self.exchange.start("QK", *_faces([Qx, Kx]), s).wait()
        _unpack([Qx, Kx], lo, 0)
        _unpack([Qx, Kx], hi, s.depth + 1)
        # halo queries compute against a partial window; their rows are
        # replaced by the owners' values before the backward reads them
        SFx, saved_x = self.be.forward(Qx, Kx, B, s.ext_dims)
        if hasattr(self.be, "check"):
            try:
                self.be.check(s.ext_dims)
            except Exception as e:  # report the global position
                pos = getattr(e, "position", None)
                if pos is not None and pos[2] >= 0:
                    e.position = (pos[0], pos[1], pos[2] - 1 + s.z0, pos[3])
                raise
        self._saved = (Qx, Kx, B, SFx, saved_x, False)
        return SFx[:, 1:-1]

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
        Qx, Kx, SFx, savedx = Q, K, SF, saved
        gSFx = self._stage("gSF", gSF)  # halo rows zero: the query-side pass's input
        names = [SFx, savedx, gSFx]
        pending = self.exchange.start("SF", *_faces(names), s)
        gB = torch.zeros_like(B)
        gQx = self.be.backward_queries(Qx, Kx, B, SFx, savedx, gSFx, s.ext_dims, gB)
        lo, hi = pending.wait()
        D = s.depth
        for plane, recv in ((0, lo), (D + 1, hi)):
            if recv is not None:
                _unpack(names, recv, plane)
            else:  # global boundary: phantom sources of zero weight
                SFx[:, plane].zero_()
                savedx[:, plane].fill_(self.be.saved_fill)
        gKx = self.be.backward_keys(Qx, Kx, B, SFx, savedx, gSFx, s.ext_dims)
        gSFx[:, 0].zero_()
        gSFx[:, D + 1].zero_()
        if s.world > 1:
            self.all_reduce(gB)
        return gQx[:, 1:-1], gKx[:, 1:-1], gB


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


def exchange_planes(x: torch.Tensor, sl: Slab, R: int, out: torch.Tensor, group=None):
    """Fill `out` {C, hi-lo, w, h} with the global planes [lo, hi) =
    [z0-R, z1+R) (clipped) of a {C, depth, w, h} slab-local tensor: this
    rank's planes by one copy, the others received from their owners straight
    into `out` (one message per channel plane run: no staging buffers)."""
    ranges = split(sl.l, sl.world)
    lo, hi = _need(sl, sl.z0, sl.z1, R)
    out[:, sl.z0 - lo:sl.z1 - lo].copy_(x)
    ops_list = []
    for q, (a, b) in enumerate(ranges):
        if q == sl.rank:
            continue
        qlo, qhi = _need(sl, a, b, R)
        s0, s1 = max(sl.z0, qlo), min(sl.z1, qhi)  # mine, needed by q
        if s0 < s1:
            for c in range(x.shape[0]):
                ops_list.append(dist.P2POp(dist.isend, x[c, s0 - sl.z0:s1 - sl.z0], q, group))
        r0, r1 = max(a, lo), min(b, hi)  # q's, needed by me
        if r0 < r1:
            for c in range(x.shape[0]):
                ops_list.append(dist.P2POp(dist.irecv, out[c, r0 - lo:r1 - lo], q, group))
    _p2p(ops_list)
    return out


def reduce_planes(contrib: torch.Tensor, sl: Slab, R: int, group=None) -> torch.Tensor:
    """contrib: this rank's additions to the global planes [z0-R, z1+R)
    (clipped).  Returns this rank's planes summed over all ranks' additions,
    in rank order."""
    ranges = split(sl.l, sl.world)
    lo, hi = _need(sl, sl.z0, sl.z1, R)
    C = contrib.shape[0]
    ops_list, recvd = [], {}
    for q, (a, b) in enumerate(ranges):
        if q == sl.rank:
            continue
        s0, s1 = max(a, lo), min(b, hi)  # my additions to q's planes
        if s0 < s1:
            for c in range(C):
                ops_list.append(dist.P2POp(dist.isend, contrib[c, s0 - lo:s1 - lo], q, group))
        qlo, qhi = _need(sl, a, b, R)
        r0, r1 = max(sl.z0, qlo), min(sl.z1, qhi)  # q's additions to mine
        if r0 < r1:
            t = torch.empty(C, r1 - r0, sl.w, sl.h, dtype=contrib.dtype, device=contrib.device)
            recvd[q] = (t, r0)
            for c in range(C):
                ops_list.append(dist.P2POp(dist.irecv, t[c], q, group))
    _p2p(ops_list)
    out = torch.zeros(C, sl.depth, sl.w, sl.h, dtype=contrib.dtype, device=contrib.device)
    for q in range(sl.world):  # fixed order
        if q == sl.rank:
            out += contrib[:, sl.z0 - lo:sl.z1 - lo]
        elif q in recvd:
            t, r0 = recvd[q]
            out[:, r0 - sl.z0:r0 - sl.z0 + t.shape[1]] += t
    return out


class CudaWarp:
    """Product backend: libmdg's depth-slab warp kernels (mdg_warp_fwd_slab /
    mdg_warp_bwd_slab): `win` holds the input planes [zi0, zi1) only, field /
    out / gout / gfield the slab's planes [z0, z1) only."""

    def fwd_whole(self, vol, field, out, dims):
        from . import ops

        n = ops.voxel_count(dims)
        P = ops._ptr
        ops._check(ops._capi.lib().mdg_warp_fwd_range(P(vol), vol.shape[0], ops.dims3(dims),
                                                      P(field), P(out), 0, n, ops._stream()))

    def bwd_whole(self, vol, field, gout, gin, gfield, dims):
        from . import ops

        n = ops.voxel_count(dims)
        P = ops._ptr
        ops._check(ops._capi.lib().mdg_warp_bwd_range(P(vol), vol.shape[0], ops.dims3(dims),
                                                      P(field), P(gout), P(gin), P(gfield), 0,
                                                      n, ops._stream()))

    def fwd_slab(self, win, field, out, dims, zi0, zi1, z0, z1):
        from . import ops

        P = ops._ptr
        ops._check(ops._capi.lib().mdg_warp_fwd_slab(P(win), win.shape[0], ops.dims3(dims),
                                                     zi0, zi1, P(field), P(out), z0, z1,
                                                     ops._stream()))

    def bwd_slab(self, win, field, gout, gin_win, gfield, dims, zi0, zi1, z0, z1):
        from . import ops

        P = ops._ptr
        ops._check(ops._capi.lib().mdg_warp_bwd_slab(P(win), win.shape[0], ops.dims3(dims),
                                                     zi0, zi1, P(field), P(gout), P(gin_win),
                                                     P(gfield), z0, z1, ops._stream()))


class SlabWarp:
    """Trilinear warp forward/backward on this rank's z-slab.  in {C, depth,
    w, h}, field {3, depth, w, h} (this rank's voxels' displacements, global
    voxel units); forward returns the rank's warped planes, backward (of the
    last forward) the rank's gin and gfield (fresh, not accumulated).

    Memory: one window buffer of the planes [z0-R, z1+R) per input (no
    full-volume buffers); the field, out, gout and gfield are the caller's
    slab-sized tensors, used in place."""

    def __init__(self, slab: Slab, backend=None, group=None, exchange=None, reduce=None,
                 all_reduce_max=None):
        self.slab = slab
        self.be = backend if backend is not None else CudaWarp()
        self.group = group
        # exchange(name, x, slab, R, out): fill out with the planes [lo, hi)
        self.exchange = exchange or (
            lambda name, x, sl, R, out: exchange_planes(x, sl, R, out, group))
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
        self._win = None

    def _window(self, C, depth, ref):
        """persistent input window, regrown when the reach grows"""
        s = self.slab
        w = self._win
        if w is None or w.shape[0] != C or w.shape[1] < depth or w.dtype != ref.dtype or \
                w.device != ref.device:
            w = torch.empty(C, depth, s.w, s.h, dtype=ref.dtype, device=ref.device)
            self._win = w
        return w[:, :depth]

    def forward(self, vol, field):
        s = self.slab
        dims = (s.h, s.w, s.l)
        if s.world == 1 and isinstance(self.be, CudaWarp):
            # one slab = the whole volume: the whole-volume kernels directly
            out = torch.empty_like(vol)
            self.be.fwd_whole(vol, field, out, dims)
            self._saved = (vol, field, None)
            return out
        R = self.all_reduce_max(warp_reach(field, s.l))
        lo, hi = _need(s, s.z0, s.z1, R)
        win = self.exchange("in", vol, s, R, self._window(vol.shape[0], hi - lo, vol))
        out = torch.empty_like(vol)
        self.be.fwd_slab(win, field, out, dims, lo, hi, s.z0, s.z1)
        self._saved = (win, field, R)
        return out

    def backward_local(self, gout):
        """(this rank's gin additions to planes [z0-R, z1+R), its gfield)"""
        if self._saved is None:
            raise RuntimeError("slab: backward without forward")
        win, field, R = self._saved
        s = self.slab
        dims = (s.h, s.w, s.l)
        gfield = torch.zeros_like(field)
        gin = torch.zeros_like(win)
        if R is None:  # world == 1: whole-volume kernels on the caller's tensors
            self.be.bwd_whole(win, field, gout, gin, gfield, dims)
            return gin, gfield
        lo, hi = _need(s, s.z0, s.z1, R)
        self.be.bwd_slab(win, field, gout, gin, gfield, dims, lo, hi, s.z0, s.z1)
        return gin, gfield

    def backward(self, gout):
        contrib, gfield = self.backward_local(gout)
        if self._saved[2] is None:  # world == 1: contrib is the whole gin
            return contrib, gfield
        gin = self.reduce("gin", contrib, self.slab, self._saved[2])
        return gin, gfield
