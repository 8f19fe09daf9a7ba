"""Depth-slab pairwise optimisation: the whole PO iteration of one pair split
along z across ranks (BASELINE config 3: "50 iterations at
160x192x224, 1/2/4/8 GPUs via depth-slab halo exchange").

Every rank owns the planes [z0, z1) of the full-resolution grid and the
matching planes of every coarser level (z0, z1 multiples of 16, so the five
levels split without remainder).  The model's ops decompose as follows
(reference files cited per op):

* conv3 (encoder conv blocks, encoder.hpp:87-91; RegHead, reghead.hpp:42-47):
  libmdg's conv over the slab, plus the neighbours' face planes' taps added
  to the two boundary output planes; the adjoint returns the face planes'
  input gradient to their owners.
* instance norm (ops.hpp:162-221): per-channel sums all-reduced (mean, then
  the centred second moment), so every rank normalises with the global
  statistics; the backward's sums are all-reduced by the same function.
* leaky ReLU, 2x average pooling, the Q/K projection + layer norm
  (attention.hpp:351-356): voxel-local.
* the ModeT operator (attention.hpp:83-166, 282-316): 1-plane Q/K halos; the
  fused kernels over the extended slab; the halo keys' gradient goes back to
  their owners.
* upsample of the running field (sampling.hpp:225-262): 1-plane halo,
  edge-replicated at the global boundary (the reference clamps there; the
  replicated plane interpolates to exactly the same value).
* warps and the composition (sampling.hpp:123-167, ops.hpp:295-298): the
  reach R = ceil(max |phi_z|) + 1 all-reduced with MAX, the planes
  [z0-R, z1+R) gathered from their owners into a window, libmdg's slab warp
  kernels (mdg_warp_fwd_slab / _bwd_slab); the scattered input gradient's
  contributions to other ranks' planes are sent back and summed in rank
  order.
* the loss (objective.hpp:39-78): NCC box sums with 4-plane halos of the
  fixed and warped images (and of the in-bounds counts), grad_reg with the
  next plane; the per-rank partial sums over owned voxels add up to the
  global means.
* parameter gradients: one all-reduce of the flat 75-tensor gradient buffer,
  then the same Adam update on every rank (replicated parameters).

The graph is recorded by torch.autograd over these functions (PyTorch is the
plumbing here: tape, device memory, torch.distributed); every convolution,
projection, attention, warp, upsample, pooling, instance norm (+ leaky ReLU)
and NCC box-sum statistic runs in libmdg; grad_reg's forward differences
(3 channels, one pass) are torch elementwise ops.  NCCL moves device tensors directly;
with gloo (the CPU tests, or several ranks sharing one GPU) the messages are
staged through host memory.  Parity: tests/test_slab_po.py (the loss and all
75 gradients against the single-volume native model)."""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops

UNIT = 16  # z split granularity: 2^(levels-1)


# --------------------------------------------------------------- plumbing
class Comm:
    """Rank, world and the point-to-point / all-reduce plumbing of one slab
    group (the default process group)."""

    def __init__(self):
        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(), dist.get_rank()
            self.staged = self.world > 1 and dist.get_backend() == "gloo"
        else:
            self.world, self.rank, self.staged = 1, 0, False

    def exchange(self, sends, recvs):
        """sends [(tensor, peer)], recvs [(tensor, peer)]: the received
        messages are written into the recv tensors (views allowed)."""
        if not sends and not recvs:
            return
        ops_, keep, back = [], [], []
        for t, q in sends:
            m = t.contiguous()
            if self.staged and m.is_cuda:
                m = m.cpu()
            keep.append(m)
            ops_.append(dist.P2POp(dist.isend, m, q))
        for t, q in recvs:
            if (self.staged and t.is_cuda) or not t.is_contiguous():
                m = torch.empty(t.shape, dtype=t.dtype, device="cpu" if self.staged else t.device)
                back.append((t, m))
            else:
                m = t
            ops_.append(dist.P2POp(dist.irecv, m, q))
        for r in dist.batch_isend_irecv(ops_):
            r.wait()
        for t, m in back:
            t.copy_(m)

    def all_reduce(self, t, op=None):
        """in place, sum (or op) over ranks"""
        if self.world == 1:
            return t
        op = dist.ReduceOp.SUM if op is None else op
        if self.staged and t.is_cuda:
            c = t.cpu()
            dist.all_reduce(c, op=op)
            t.copy_(c)
        else:
            dist.all_reduce(t, op=op)
        return t

    def all_reduce_max_int(self, v: int) -> int:
        if self.world == 1:
            return v
        t = torch.tensor([v], dtype=torch.int64)
        if not self.staged:
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return int(t.item())


def split_units(l: int, world: int):
    """Balanced z ranges [(z0, z1)] in whole units of 16 planes."""
    if l % UNIT:
        raise ops.InvalidInput(f"slab PO: depth {l} must be a multiple of {UNIT}")
    units = l // UNIT
    if units < world:
        raise ops.InvalidInput(f"slab PO: {units} units of {UNIT} planes for {world} ranks")
    base, rem = divmod(units, world)
    out, z = [], 0
    for r in range(world):
        n = (base + (1 if r < rem else 0)) * UNIT
        out.append((z, z + n))
        z += n
    return out


class Geom:
    """Global dims (h, w, l) of the full-resolution grid and this rank's
    z range; level e (0 = full resolution) divides everything by 2^e.

    reach None: every warp all-reduces its data-dependent reach (a host
    round trip per warp).  reach R: the warps exchange R planes per side
    without looking at the field, a field that samples further is flagged on
    the device (err) and reported after the step — no host round trip
    inside the step, so it can be captured as one CUDA graph."""

    def __init__(self, dims, comm: Comm, reach=None):
        self.dims = tuple(int(v) for v in dims)
        self.comm = comm
        self.ranges = split_units(self.dims[2], comm.world)
        self.z0, self.z1 = self.ranges[comm.rank]
        self.reach = None if reach is None else int(reach)
        self.err = None  # device int32 word of the fixed-reach mode
        self.defer_checks = self.reach is not None

    def level(self, e):
        """(dims, z0, z1, all ranks' ranges) of level e; dims halve rounding
        up (common.hpp:72-74 halved), z exactly (multiples of 16)"""
        h, w, l = self.dims
        for _ in range(e):
            h, w, l = (h + 1) // 2, (w + 1) // 2, (l + 1) // 2
        return (h, w, l), self.z0 >> e, self.z1 >> e, \
            [(a >> e, b >> e) for a, b in self.ranges]


# ------------------------------------------------------ autograd functions
class _Halo(torch.autograd.Function):
    """x {C, D, w, h} -> {C, D+2k, w, h} with the neighbours' k face planes;
    zero (or, edge=True, the boundary plane repeated) at the global
    boundary.  Backward: the halo planes' gradient goes back to the owners."""

    @staticmethod
    def forward(ctx, x, k, edge, comm):
        C, D, W, H = x.shape
        if D < k:
            raise ops.InvalidInput(f"slab PO: {D} planes per rank < halo {k}")
        out = x.new_empty(C, D + 2 * k, W, H)
        out[:, k:k + D] = x
        r, n = comm.rank, comm.world
        if r == 0 and not edge:  # global boundary: zero padding
            out[:, :k].zero_()
        if r == n - 1 and not edge:
            out[:, D + k:].zero_()
        sends, recvs = [], []
        if r > 0:
            sends.append((x[:, :k], r - 1))
            recvs.append((out[:, :k], r - 1))
        if r < n - 1:
            sends.append((x[:, D - k:], r + 1))
            recvs.append((out[:, D + k:], r + 1))
        comm.exchange(sends, recvs)
        if edge:
            if r == 0:
                out[:, :k] = x[:, :1]
            if r == n - 1:
                out[:, D + k:] = x[:, D - 1:D]
        ctx.k, ctx.edge, ctx.comm, ctx.D = k, edge, comm, D
        return out

    @staticmethod
    def backward(ctx, g):
        k, D, comm = ctx.k, ctx.D, ctx.comm
        r, n = comm.rank, comm.world
        gx = g[:, k:k + D].clone()
        sends, recvs, got = [], [], []
        if r > 0:
            sends.append((g[:, :k], r - 1))
            t = torch.empty_like(gx[:, :k])
            recvs.append((t, r - 1))
            got.append((t, 0))
        if r < n - 1:
            sends.append((g[:, D + k:], r + 1))
            t = torch.empty_like(gx[:, :k])
            recvs.append((t, r + 1))
            got.append((t, D - k))
        comm.exchange(sends, recvs)
        for t, z in got:
            gx[:, z:z + k] += t
        if ctx.edge:
            if r == 0:
                gx[:, 0] += g[:, :k].sum(1)
            if r == n - 1:
                gx[:, D - 1] += g[:, D + k:].sum(1)
        return gx, None, None, None


def halo(x, k, comm, edge=False):
    return _Halo.apply(x, k, edge, comm)


class _AllReduce(torch.autograd.Function):
    """sum over ranks; the adjoint of a replicated sum is the sum of the
    ranks' gradients"""

    @staticmethod
    def forward(ctx, t, comm):
        ctx.comm = comm
        return comm.all_reduce(t.clone())

    @staticmethod
    def backward(ctx, g):
        return ctx.comm.all_reduce(g.clone()), None


def all_reduce(t, comm):
    return _AllReduce.apply(t, comm)


def _dims_of(x):  # {C, l, w, h} -> (h, w, l)
    return (x.shape[3], x.shape[2], x.shape[1])


def _conv3(x, w, b, out):
    """libmdg's 3x3x3 conv (mdg_encoder_conv3_fwd) of {ic, D, w, h}, zero
    padded at its own faces; b nullable"""
    ic, D, W, H = x.shape
    ops._check(ops._capi.lib().mdg_encoder_conv3_fwd(ops._ptr(x), ic, ops.dims3((H, W, D)),
                                                     ops._ptr(w), ops._ptr(b), w.shape[0],
                                                     ops._ptr(out), ops._stream()))
    return out


def _conv3_bwd(x, w, g, gin, gw, gb):
    """mdg_encoder_conv3_bwd: accumulates gin, gw, gb (each nullable)"""
    ic, D, W, H = x.shape
    ops._check(ops._capi.lib().mdg_encoder_conv3_bwd(ops._ptr(x), ic, ops.dims3((H, W, D)),
                                                     ops._ptr(w), w.shape[0], ops._ptr(g),
                                                     ops._ptr(gin), ops._ptr(gw), ops._ptr(gb),
                                                     ops._stream()))


class _Conv3Slab(torch.autograd.Function):
    """conv3 of a slab {ic, D, w, h}, zero padded at the global z faces.
    libmdg's conv runs over the slab itself (zero padded at the slab's own
    faces, output contiguous: no extended copy, no interior slice); the
    neighbours' face planes then add their dz = -1 / +1 taps to the two
    boundary output planes (a conv over the 2-plane volume [face, 0] or
    [0, face], no bias).  Backward: the slab's conv backward, plus each face
    plane's share of the kernel gradient and its input gradient, which goes
    back to the owner.  One rank: libmdg's conv alone."""

    @staticmethod
    def forward(ctx, x, w, b, comm):
        x = x.contiguous()
        ic, D, W, H = x.shape
        oc = w.shape[0]
        out = _conv3(x, w, b, x.new_empty(oc, D, W, H))
        r, n = comm.rank, comm.world
        lo = hi = None
        if n > 1:
            sends, recvs = [], []
            if r > 0:  # [rank r-1's last plane, 0]
                lo = x.new_zeros(ic, 2, W, H)
                sends.append((x[:, :1], r - 1))
                recvs.append((lo[:, :1], r - 1))
            if r < n - 1:  # [0, rank r+1's first plane]
                hi = x.new_zeros(ic, 2, W, H)
                sends.append((x[:, D - 1:], r + 1))
                recvs.append((hi[:, 1:], r + 1))
            comm.exchange(sends, recvs)
            if lo is not None:
                out[:, 0] += _conv3(lo, w, None, x.new_empty(oc, 2, W, H))[:, 1]
            if hi is not None:
                out[:, D - 1] += _conv3(hi, w, None, x.new_empty(oc, 2, W, H))[:, 0]
        ctx.save_for_backward(x, w, lo, hi)
        ctx.comm = comm
        return out

    @staticmethod
    def backward(ctx, g):
        x, w, lo, hi = ctx.saved_tensors
        comm = ctx.comm
        r = comm.rank
        g = g.contiguous()
        ic, D, W, H = x.shape
        oc = w.shape[0]
        gin, gw, gb = torch.zeros_like(x), torch.zeros_like(w), w.new_zeros(oc)
        _conv3_bwd(x, w, g, gin, gw, gb)
        sends, recvs, got = [], [], []
        if lo is not None:
            gm = g.new_zeros(oc, 2, W, H)
            gm[:, 1] = g[:, 0]
            gl = torch.zeros_like(lo)
            _conv3_bwd(lo, w, gm, gl, gw, None)
            sends.append((gl[:, :1], r - 1))
            t = x.new_empty(ic, 1, W, H)
            recvs.append((t, r - 1))
            got.append((t, 0))
        if hi is not None:
            gm = g.new_zeros(oc, 2, W, H)
            gm[:, 0] = g[:, D - 1]
            gh = torch.zeros_like(hi)
            _conv3_bwd(hi, w, gm, gh, gw, None)
            sends.append((gh[:, 1:], r + 1))
            t = x.new_empty(ic, 1, W, H)
            recvs.append((t, r + 1))
            got.append((t, D - 1))
        comm.exchange(sends, recvs)
        for t, z in got:
            gin[:, z:z + 1] += t
        return gin, gw, gb, None


def conv3_slab(x, w, b, comm):
    """zero-padded conv3 of a slab (encoder.hpp:87-91, reghead.hpp:42-47)"""
    return _Conv3Slab.apply(x, w, b, comm)


class _Project(torch.autograd.Function):
    """op_project_qk (attention.hpp:351-356) -> planar Q, K {K, n}"""

    @staticmethod
    def forward(ctx, f, m, W, b, g, beta):
        f2, m2 = f.reshape(f.shape[0], -1).contiguous(), m.reshape(m.shape[0], -1).contiguous()
        p = ops.ProjectionParams(W, b, g, beta)
        Q, K = ops.project_qk(f2, m2, p, layout=ops.MDG_QK_PLANAR)
        ctx.save_for_backward(f2, m2, W, b, g, beta)
        ctx.shape = f.shape
        return Q, K

    @staticmethod
    def backward(ctx, gQ, gK):
        f2, m2, W, b, g, beta = ctx.saved_tensors
        zero = f2.new_zeros(W.shape[0], f2.shape[1])
        gQ = zero if gQ is None else gQ
        gK = zero if gK is None else gK
        gf, gm, gp = ops.project_qk_bwd(f2, m2, ops.ProjectionParams(W, b, g, beta),
                                        gQ.contiguous(), gK.contiguous(),
                                        layout=ops.MDG_QK_PLANAR)
        return (gf.view(ctx.shape), gm.view(ctx.shape), gp.weight, gp.bias, gp.ln_gamma,
                gp.ln_beta)


class _ModeT(torch.autograd.Function):
    """the fused ModeT operator (na_fused + subfields) on extended planar
    Q/K {S*d, D+2, w, h}; the numeric check reports global positions"""

    @staticmethod
    def forward(ctx, Qx, Kx, B, S, hd, z_shift, defer=False):
        d = _dims_of(Qx)
        cfg = ops.AttentionConfig(S, hd, 3)
        Q2, K2 = Qx.reshape(S * hd, -1).contiguous(), Kx.reshape(S * hd, -1).contiguous()
        SF, LSE = ops.modet_fwd(Q2, K2, B.contiguous(), d, cfg, layout=ops.MDG_QK_PLANAR,
                                check=False)
        try:
            if not defer:  # else the stream's flag is read once after the step
                ops.check_numeric(d)
        except ops.NumericError as e:
            pos = getattr(e, "position", None)
            if pos is not None and pos[2] >= 0:
                e.position = (pos[0], pos[1], pos[2] + z_shift, pos[3])
            raise
        ctx.save_for_backward(Q2, K2, B, SF, LSE)
        ctx.cfg, ctx.d = cfg, d
        return SF.view(3 * S, *Qx.shape[1:])

    @staticmethod
    def backward(ctx, gSF):
        Q2, K2, B, SF, LSE = ctx.saved_tensors
        gQ, gK, gB = ops.modet_bwd(Q2, K2, B, SF, LSE, gSF.reshape(SF.shape).contiguous(), ctx.d,
                                   ctx.cfg, layout=ops.MDG_QK_PLANAR)
        shp = (Q2.shape[0], *gSF.shape[1:])
        return gQ.view(shp), gK.view(shp), gB, None, None, None, None


class _Upsample(torch.autograd.Function):
    """op_upsample_field_2x on an extended coarse slab (values x2) onto
    (h, w) = the finer level's, z doubled"""

    @staticmethod
    def forward(ctx, x, hw):
        d = _dims_of(x)
        target = (hw[0], hw[1], 2 * d[2])
        ctx.d, ctx.t = d, target
        return ops.upsample_field_2x(x.contiguous(), target, d)

    @staticmethod
    def backward(ctx, g):
        return ops.upsample_field_2x_bwd(g.contiguous(), ctx.d, ctx.t), None


def upsample_slab(phi_c, comm, hw):
    """coarse slab {3, Dc, wc, hc} -> fine slab {3, 2Dc, 2wc, 2hc}: fine plane
    z samples coarse z/2, so the coarse slab needs its next plane (edge-
    replicated at the global end, where the reference clamps).  One rank:
    the whole volume, upsampled directly."""
    Dc = phi_c.shape[1]
    if comm.world == 1:
        return _Upsample.apply(phi_c, hw)
    return _Upsample.apply(halo(phi_c, 1, comm, edge=True), hw)[:, 2:2 + 2 * Dc]


def warp_reach(field_local, l):
    fz = field_local[2]
    if fz.numel() == 0:
        return 1
    if not bool(torch.isfinite(fz).all()):
        return l
    return min(l, int(torch.ceil(fz.abs().max()).item()) + 1)


class _Warp(torch.autograd.Function):
    """op_warp of a slab {C, D, w, h} by its field {3, D, w, h} (global voxel
    units): the input planes within the all-reduced reach are gathered into a
    window, the slab kernels index it directly."""

    @staticmethod
    def forward(ctx, vol, field, geom, e):
        comm = geom.comm
        (h, w, l), z0, z1, ranges = geom.level(e)
        R = geom.reach if geom.reach is not None else \
            comm.all_reduce_max_int(warp_reach(field, l))
        need = [(max(0, a - R), min(l, b + R)) for a, b in ranges]
        lo, hi = need[comm.rank]
        vol = vol.contiguous()
        C = vol.shape[0]
        if (lo, hi) == (z0, z1):  # the window is the slab itself (one rank)
            win = vol
        else:
            win = vol.new_empty(C, hi - lo, w, h)
            win[:, z0 - lo:z1 - lo] = vol
        sends, recvs = [], []
        for q, (a, b) in enumerate(ranges):
            if q == comm.rank:
                continue
            s0, s1 = max(z0, need[q][0]), min(z1, need[q][1])  # mine, needed by q
            if s0 < s1:
                sends.append((vol[:, s0 - z0:s1 - z0], q))
            r0, r1 = max(a, lo), min(b, hi)  # q's, needed by me
            if r0 < r1:
                recvs.append((win[:, r0 - lo:r1 - lo], q))
        comm.exchange(sends, recvs)
        field = field.contiguous()
        out = torch.empty_like(vol)
        L, P = ops._capi.lib(), ops._ptr
        if geom.err is not None:
            ops._check(L.mdg_warp_fwd_slab_async(P(win), C, ops.dims3((h, w, l)), lo, hi,
                                                 P(field), P(out), z0, z1, geom.err.data_ptr(),
                                                 ops._stream()))
        else:
            ops._check(L.mdg_warp_fwd_slab(P(win), C, ops.dims3((h, w, l)), lo, hi, P(field),
                                           P(out), z0, z1, ops._stream()))
        ctx.save_for_backward(win, field)
        ctx.geom, ctx.e, ctx.need = geom, e, need
        return out

    @staticmethod
    def backward(ctx, gout):
        win, field = ctx.saved_tensors
        geom, need = ctx.geom, ctx.need
        comm = geom.comm
        (h, w, l), z0, z1, ranges = geom.level(ctx.e)
        lo, hi = need[comm.rank]
        C = win.shape[0]
        gin_w = torch.zeros_like(win)
        gfield = torch.zeros_like(field)
        L, P = ops._capi.lib(), ops._ptr
        if geom.err is not None:
            ops._check(L.mdg_warp_bwd_slab_async(P(win), C, ops.dims3((h, w, l)), lo, hi,
                                                 P(field), P(gout.contiguous()), P(gin_w),
                                                 P(gfield), z0, z1, geom.err.data_ptr(),
                                                 ops._stream()))
        else:
            ops._check(L.mdg_warp_bwd_slab(P(win), C, ops.dims3((h, w, l)), lo, hi, P(field),
                                           P(gout.contiguous()), P(gin_w), P(gfield), z0, z1,
                                           ops._stream()))
        # contributions to other ranks' planes go back to their owners,
        # summed there in rank order
        sends, recvs, got = [], [], {}
        for q, (a, b) in enumerate(ranges):
            if q == comm.rank:
                continue
            s0, s1 = max(a, lo), min(b, hi)  # my additions to q's planes
            if s0 < s1:
                sends.append((gin_w[:, s0 - lo:s1 - lo], q))
            r0, r1 = max(z0, need[q][0]), min(z1, need[q][1])  # q's additions to mine
            if r0 < r1:
                t = win.new_empty(C, r1 - r0, w, h)
                recvs.append((t, q))
                got[q] = (t, r0)
        comm.exchange(sends, recvs)
        if (lo, hi) == (z0, z1) and not got:  # nothing to or from other ranks
            return gin_w, gfield, None, None
        gin = win.new_zeros(C, z1 - z0, w, h)
        for q in range(comm.world):
            if q == comm.rank:
                gin += gin_w[:, z0 - lo:z1 - lo]
            elif q in got:
                t, r0 = got[q]
                gin[:, r0 - z0:r0 - z0 + t.shape[1]] += t
        return gin, gfield, None, None


def warp_slab(vol, field, geom, e):
    return _Warp.apply(vol, field, geom, e)


def _dptr(t):
    """pointer of a contiguous float64 device tensor (the fp64 sums)"""
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise ops.InvalidInput("slab PO: fp64 sums must be contiguous float64")
    return t.data_ptr()


class _InLrelu(torch.autograd.Function):
    """lrelu(instance_norm(x)) of a slab (ops.hpp:162-238) by libmdg's
    encoder kernels, the per-channel sums all-reduced between the passes
    (mean, then the centred second moment; backward: sum gy, sum gy xh),
    accumulated in fp64 so the ranks' grouping costs no accuracy.
    The gamma / beta gradients returned are this slab's share (the
    parameter-gradient all-reduce adds the ranks')."""

    @staticmethod
    def forward(ctx, x, g, b, slope, n_global, comm):
        x = x.contiguous()
        C, n = x.shape[0], x[0].numel()
        L, P, st = ops._capi.lib(), ops._ptr, ops._stream()
        s1 = x.new_empty(C, dtype=torch.float64)
        ops._check(L.mdg_in_slab_sums(P(x), C, n, None, _dptr(s1), st))
        mean = (comm.all_reduce(s1) / n_global).float()
        s2 = x.new_empty(C, dtype=torch.float64)
        ops._check(L.mdg_in_slab_sums(P(x), C, n, P(mean), _dptr(s2), st))
        inv = (1.0 / torch.sqrt(comm.all_reduce(s2) / n_global + 1e-5)).float()
        z = torch.empty_like(x)
        ops._check(L.mdg_in_lrelu_apply(P(x), C, n, P(mean), P(inv), P(g), P(b), float(slope),
                                        P(z), st))
        ctx.save_for_backward(x, g, b, mean, inv)
        ctx.slope, ctx.n_global, ctx.comm = float(slope), n_global, comm
        return z

    @staticmethod
    def backward(ctx, gz):
        x, g, b, mean, inv = ctx.saved_tensors
        gz = gz.contiguous()
        C, n = x.shape[0], x[0].numel()
        L, P, st = ops._capi.lib(), ops._ptr, ops._stream()
        sums = x.new_empty(C, 2, dtype=torch.float64)
        ops._check(L.mdg_in_lrelu_bwd_sums(P(x), P(gz), C, n, P(mean), P(inv), P(g), P(b),
                                           ctx.slope, _dptr(sums), st))
        local = sums.float()
        sums = ctx.comm.all_reduce(sums).float()
        gx = torch.empty_like(x)
        ops._check(L.mdg_in_lrelu_bwd_apply(P(x), P(gz), C, n, P(mean), P(inv), P(g), P(b),
                                            ctx.slope, P(sums), ctx.n_global, P(gx), st))
        return gx, local[:, 1].contiguous(), local[:, 0].contiguous(), None, None, None


class _AvgPool(torch.autograd.Function):
    """2x average pooling (sampling.hpp:171-219) of a slab: z even per rank,
    odd x / y extents repeat their last voxel as in the reference"""

    @staticmethod
    def forward(ctx, x):
        x = x.contiguous()
        C, D, W, H = x.shape
        out = x.new_empty(C, (D + 1) // 2, (W + 1) // 2, (H + 1) // 2)
        L, P = ops._capi.lib(), ops._ptr
        ops._check(L.mdg_avgpool2_fwd(P(x), C, ops.dims3((H, W, D)), P(out), ops._stream()))
        ctx.shape = x.shape
        return out

    @staticmethod
    def backward(ctx, g):
        C, D, W, H = ctx.shape
        gin = g.new_zeros(ctx.shape)
        L, P = ops._capi.lib(), ops._ptr
        ops._check(L.mdg_avgpool2_bwd(P(g.contiguous()), C, ops.dims3((H, W, D)), P(gin),
                                      ops._stream()))
        return gin


# ------------------------------------------------------------- the model
def conv_block(x, p, geom, e, slope):
    """op_conv_block (encoder.hpp:87-91); p = (w1, b1, g1, beta1, w2, b2,
    g2, beta2)"""
    (h, w, l), _, _, _ = geom.level(e)
    n = h * w * l
    comm = geom.comm
    for wk, bk, gk, btk in (p[0:4], p[4:8]):
        x = _InLrelu.apply(conv3_slab(x, wk, bk, comm), gk, btk, slope, n, comm)
    return x


def encode(image, blocks, geom, slope):
    """op_encode (encoder.hpp:102-116): features fine -> coarse"""
    feats = []
    x = conv_block(image, blocks[0], geom, 0, slope)
    feats.append(x)
    for e in range(1, len(blocks)):
        x = _AvgPool.apply(x)
        x = conv_block(x, blocks[e], geom, e, slope)
        feats.append(x)
    return feats


class _NccSlab(torch.autograd.Function):
    """sum of NCC's per-voxel cc over the slab's own voxels (libmdg's box-sum
    kernels on the extended grid, mdg_ncc_slab_fwd / _bwd)"""

    @staticmethod
    def forward(ctx, fx, gx, window, zv0, zv1):
        fx, gx = fx.contiguous(), gx.contiguous()
        e = ops.dims3(_dims_of(fx))
        out = fx.new_empty(1)
        L, P = ops._capi.lib(), ops._ptr
        ops._check(L.mdg_ncc_slab_fwd(P(fx), P(gx), e, window, zv0, zv1, P(out), ops._stream()))
        ctx.save_for_backward(fx, gx)
        ctx.args = (e, window, zv0, zv1)
        return out[0]

    @staticmethod
    def backward(ctx, g):
        fx, gx = ctx.saved_tensors
        e, window, zv0, zv1 = ctx.args
        gw = torch.empty_like(gx)
        L, P = ops._capi.lib(), ops._ptr
        g = g.reshape(1).contiguous()  # read on the device: no host round trip
        ops._check(L.mdg_ncc_slab_bwd_dev(P(fx), P(gx), e, window, zv0, zv1, 1.0, P(g), P(gw),
                                          ops._stream()))
        return None, gw, None, None, None


def grad_reg_slab(phi, geom):
    """op_grad_reg (ops.hpp:326-382): this slab's share (forward differences
    of its planes, the z one reaching the next slab's first plane)"""
    comm = geom.comm
    (h, w, l), _, _, _ = geom.level(0)
    n = h * w * l
    D = phi.shape[1]
    if comm.world == 1:
        u = phi
        dz = phi[:, 1:] - phi[:, :-1]
    else:
        ext = halo(phi, 1, comm)
        u = ext[:, 1:1 + D]
        dz = ext[:, 2:2 + D] - u
        if comm.rank == comm.world - 1:
            dz = dz[:, :D - 1]  # the last plane has no forward difference
    reg = 0.0
    for diff, dim in ((u[..., 1:] - u[..., :-1], h), (u[:, :, 1:] - u[:, :, :-1], w), (dz, l)):
        reg = reg + (diff * diff).sum() / float(n - n // dim)
    return reg / 3.0


def slab_loss(fixed, warped, phi, geom, lam, window):
    """op_total_loss (objective.hpp:39-78) minus the warp: this rank's part
    of ncc + lam * grad_reg (the parts add up to the global loss)"""
    comm = geom.comm
    (h, w, l), _, _, _ = geom.level(0)
    r = window // 2
    fx = halo(fixed, r, comm)
    gx = halo(warped, r, comm)
    D = fixed.shape[1]
    zv0 = r if comm.rank == 0 else 0
    zv1 = D + r if comm.rank == comm.world - 1 else D + 2 * r
    ncc = -_NccSlab.apply(fx, gx, window, zv0, zv1) / float(h * w * l)
    if lam == 0.0:
        return ncc, ncc, ncc.new_zeros(())
    reg = grad_reg_slab(phi, geom)
    return ncc + lam * reg, ncc, reg


class SlabModel:
    """The small-preset model (or any base_channels / heads / head_dim) with
    its PO iteration decomposed over depth slabs.  `tensors`: the 75
    ModelParams tensors (ops.init_model order), replicated on every rank;
    images are this rank's planes {1, z1-z0, w, h}.

    reach: None (each warp all-reduces its data-dependent reach) or a fixed
    plane count R (see Geom) — the mode po_step(..., graph=True) captures as
    one CUDA graph per iteration."""

    def __init__(self, tensors, dims, lam=1.0, window=9, slope=0.2, heads=(8, 4, 2, 1, 1),
                 head_dim=6, comm: Comm | None = None, reach=None, diffeomorphic=False,
                 ss_steps=7):
        self.comm = comm or Comm()
        self.geom = Geom(dims, self.comm, reach)
        self.params = [t.detach().clone().contiguous().requires_grad_(True) for t in tensors]
        if len(self.params) != 75:
            raise ops.InvalidInput("slab PO: expects the 75 ModelParams tensors")
        if reach is not None:
            self.geom.err = torch.zeros(1, dtype=torch.int32, device=self.params[0].device)
        self.lam, self.window, self.slope = float(lam), int(window), float(slope)
        self.heads, self.hd = tuple(heads), int(head_dim)
        self.diffeomorphic, self.ss_steps = bool(diffeomorphic), int(ss_steps)
        if self.diffeomorphic and self.ss_steps < 1:
            raise ops.InvalidInput("scaling_squaring: steps must be >= 1")
        self.opt = ops.AdamOptimizer([p.data for p in self.params])
        self.grads = [torch.zeros_like(p) for p in self.params]
        self._graph = None

    @property
    def z_range(self):
        return self.geom.z0, self.geom.z1

    def local(self, full):
        """this rank's planes of a {C, l, w, h} tensor"""
        return full[:, self.geom.z0:self.geom.z1].contiguous()

    def forward(self, fixed, moving):
        """build_pipeline (engine.hpp:179-219) on the slab: phi {3, D, w, h}"""
        P = self.params
        blocks = [P[8 * k:8 * k + 8] for k in range(5)]
        geom, comm = self.geom, self.comm
        ff = encode(fixed, blocks, geom, self.slope)
        mf = encode(moving, blocks, geom, self.slope)
        phi = phi_up = None
        for k in range(5):
            e = 4 - k
            W, b, g, beta, B, rw, rb = P[40 + 7 * k:47 + 7 * k]
            f, m = ff[e], mf[e]
            m_in = m
            if k > 0:
                (he, we, _), _, _, _ = geom.level(e)
                phi_up = upsample_slab(phi, comm, (he, we))
                m_in = warp_slab(m, phi_up, geom, e)
            S = self.heads[k]
            Q, K = _Project.apply(f, m_in, W, b, g, beta)
            shp = (S * self.hd, *f.shape[1:])
            _, z0, _, _ = geom.level(e)
            if comm.world == 1:  # the whole volume: no halo planes
                SF = _ModeT.apply(Q.view(shp), K.view(shp), B, S, self.hd, z0,
                                  geom.defer_checks)
            else:
                Qx, Kx = halo(Q.view(shp), 1, comm), halo(K.view(shp), 1, comm)
                SF = _ModeT.apply(Qx, Kx, B, S, self.hd, z0 - 1, geom.defer_checks)[:, 1:-1]
            res = conv3_slab(SF, rw, rb, comm)
            if self.diffeomorphic:
                # op_scaling_squaring (reghead.hpp:52-57): v / 2^T, then T
                # self-compositions phi + warp(phi, phi)
                res = res * (1.0 / float(1 << self.ss_steps))
                for _ in range(self.ss_steps):
                    res = res + warp_slab(res, res, geom, e)
            phi = res if k == 0 else res + warp_slab(phi_up, res, geom, e)
        return phi

    def _body(self, fixed, moving, backward):
        """forward (+ backward and the gradient all-reduce into self.grads)
        with no host round trip when the reach is fixed"""
        if self.geom.err is not None:
            self.geom.err.zero_()
        with torch.set_grad_enabled(backward):
            phi = self.forward(fixed, moving)
            warped = warp_slab(moving, phi, self.geom, 0)
            total, ncc, reg = slab_loss(fixed, warped, phi, self.geom, self.lam, self.window)
            if backward:
                total.backward()
        terms = torch.stack([total.detach(), ncc.detach(), torch.as_tensor(reg).detach()
                             .to(total.device, total.dtype)])
        self.comm.all_reduce(terms)
        if backward:
            flat = torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1)
                              for p in self.params])
            self.comm.all_reduce(flat)  # the one parameter-gradient all-reduce
            o = 0
            for g in self.grads:
                g.copy_(flat[o:o + g.numel()].view_as(g))
                o += g.numel()
        return terms, phi.detach()

    def _post_check(self):
        """the checks a fixed-reach step defers to its end"""
        if not self.geom.defer_checks:
            return
        ops.check_numeric(self.geom.dims)
        if int(self.geom.err.item()):
            raise ops.InvalidInput(f"slab PO: the field sampled beyond the fixed reach of "
                                   f"{self.geom.reach} planes; construct with a larger reach")

    def loss_step(self, fixed, moving, backward=True):
        """run_loss_step (engine.hpp:316-340): the global {total, ncc, reg}
        (identical on every rank) and this rank's phi; with backward, the
        all-reduced parameter gradients in self.grads."""
        for p in self.params:
            p.grad = None
        out = self._body(fixed, moving, backward)
        self._post_check()
        return out

    def _replay(self, fixed, moving):
        """the loss step as one CUDA graph (captured on first use; the images
        are copied into the graph's static inputs)"""
        if self._graph is None:
            if self.geom.reach is None:
                raise ops.InvalidInput("slab PO: graph mode needs a fixed reach")
            if self.comm.staged:
                raise ops.InvalidInput("slab PO: graph mode needs NCCL (or one rank)")
            self._sf, self._sm = fixed.clone(), moving.clone()
            for p in self.params:
                p.grad = torch.zeros_like(p)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for _ in range(2):  # warm-up (allocator, autograd, tensor maps)
                    for p in self.params:
                        p.grad.zero_()
                    self._body(self._sf, self._sm, True)
            torch.cuda.current_stream().wait_stream(side)
            self._graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self._graph):
                for p in self.params:
                    p.grad.zero_()
                self._gout = self._body(self._sf, self._sm, True)
        if fixed.data_ptr() != self._sf.data_ptr():
            self._sf.copy_(fixed)
        if moving.data_ptr() != self._sm.data_ptr():
            self._sm.copy_(moving)
        self._graph.replay()
        self._post_check()
        return self._gout[0].clone(), self._gout[1].clone()

    def po_step(self, fixed, moving, lr=1e-4, graph=False):
        """one pairwise_optimize iteration (engine.hpp:389-398); graph=True
        replays the loss step as a CUDA graph (fixed reach) and runs Adam
        after it"""
        if graph:
            terms, phi = self._replay(fixed, moving)
        else:
            terms, phi = self.loss_step(fixed, moving, backward=True)
        self.opt.step(lr, self.grads)
        return terms, phi
