"""Python face of the B200 ModeT hot path (torch tensors as device memory).

Mirrors the reference's interfaces so code written against mdreg reads the
same way:

* ``kern`` functions have the names, argument meaning and overwrite /
  accumulate rules of ``mdreg::kern::*`` (attention.hpp, sampling.hpp,
  ops.hpp) and take CUDA fp32 tensors in the reference layouts;
* errors raise :class:`InvalidInput` / :class:`NumericError`, the Python
  counterparts of ``mdreg::invalid_input`` / ``mdreg::numeric_error``
  (common.hpp:25-37);
* the fused ModeT operator (``modet_fwd`` / ``modet_bwd``) is the B200-native
  replacement of ``op_na_fused`` + ``op_subfields``.

Everything runs on the current torch CUDA stream through ``libmdg.so``; there
is no CPU path.  torch provides memory and streams only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _capi
from ._capi import MDG_QK_PLANAR, MDG_QK_POSMAJOR, Dims3


class InvalidInput(ValueError):
    """mdreg::invalid_input — bad arguments or inconsistent shapes."""


class NumericError(RuntimeError):
    """mdreg::numeric_error — non-finite values during computation."""

    position = None  # (x, y, z, head) for attention errors


class ParseError(RuntimeError):
    """mdreg::parse_error — malformed or truncated files (common.hpp:29-32)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside libmdg."""


def _check(status: int):
    if status == _capi.MDG_OK:
        return
    L = _capi.lib()
    msg = L.mdg_last_error().decode()
    if status == _capi.MDG_EINVAL:
        raise InvalidInput(msg)
    if status == _capi.MDG_EPARSE:
        raise ParseError(msg)
    if status == _capi.MDG_ENUMERIC:
        e = NumericError(msg)
        pos = [C.c_int() for _ in range(4)]
        L.mdg_last_error_position(*[C.byref(v) for v in pos])
        e.position = tuple(v.value for v in pos)
        raise e
    raise CudaError(msg)


def _ptr(t, name="tensor"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise InvalidInput(f"{name}: expected a torch tensor")
    if not t.is_cuda:
        raise InvalidInput(f"{name}: must be a CUDA tensor (no CPU path)")
    if t.dtype != torch.float32:
        raise InvalidInput(f"{name}: must be float32")
    if not t.is_contiguous():
        raise InvalidInput(f"{name}: must be contiguous")
    return t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def dims3(d) -> Dims3:
    h, w, l = (int(v) for v in d)
    return Dims3(h, w, l)


def voxel_count(d) -> int:
    h, w, l = d
    return int(h) * int(w) * int(l)


def halved(d):
    """common.hpp:70-74 (ceil)."""
    return tuple((int(v) + 1) // 2 for v in d)


@dataclass
class AttentionConfig:
    """attention.hpp:40-54."""

    heads: int = 1
    head_dim: int = 6
    neighborhood: int = 3

    def radius(self) -> int:
        return (self.neighborhood - 1) // 2

    def window(self) -> int:
        return self.neighborhood ** 3

    def validate(self):
        if self.neighborhood < 3 or self.neighborhood % 2 == 0:
            raise InvalidInput("attention: neighborhood must be odd and >= 3")
        if self.heads < 1 or self.head_dim < 1:
            raise InvalidInput("attention: heads and head_dim must be positive")


def window_offset(o: int, nb: int = 3):
    """attention.hpp:57-60 (evaluated by libmdg)."""
    off = (C.c_int * 3)()
    _check(_capi.lib().mdg_window_offset(o, nb, off))
    return tuple(off)


class kern:  # noqa: N801 — mirrors the reference namespace mdreg::kern
    """Reference-shaped kernel tier: in-place on caller-owned CUDA tensors."""

    @staticmethod
    def resolve_axis(x: torch.Tensor, dim: int):
        n = x.numel()
        i0 = torch.empty(n, dtype=torch.int32, device=x.device)
        i1 = torch.empty_like(i0)
        live = torch.empty_like(i0)
        f = torch.empty(n, dtype=torch.float32, device=x.device)
        _check(_capi.lib().mdg_resolve_axis(_ptr(x, "x"), n, dim, i0.data_ptr(), i1.data_ptr(),
                                            f.data_ptr(), live.data_ptr(), _stream()))
        return i0, i1, f, live

    @staticmethod
    def na_fused_fwd(Q, K, B, d, S, hd, nb, W):
        _check(_capi.lib().mdg_na_fused_fwd(_ptr(Q, "Q"), _ptr(K, "K"), _ptr(B, "B"), dims3(d),
                                            S, hd, nb, _ptr(W, "W"), _stream()))

    @staticmethod
    def na_fused_bwd(Q, K, W, d, S, hd, nb, gW, gQ, gK, gB):
        _check(_capi.lib().mdg_na_fused_bwd(_ptr(Q), _ptr(K), _ptr(W), dims3(d), S, hd, nb,
                                            _ptr(gW), _ptr(gQ), _ptr(gK), _ptr(gB), _stream()))

    @staticmethod
    def subfields_fwd(W, d, S, nb, out):
        _check(_capi.lib().mdg_subfields_fwd(_ptr(W), dims3(d), S, nb, _ptr(out), _stream()))

    @staticmethod
    def subfields_bwd(d, S, nb, gout, gW):
        _check(_capi.lib().mdg_subfields_bwd(dims3(d), S, nb, _ptr(gout), _ptr(gW), _stream()))

    @staticmethod
    def warp_fwd(in_, channels, d, field, out):
        _check(_capi.lib().mdg_warp_fwd(_ptr(in_), channels, dims3(d), _ptr(field), _ptr(out),
                                        _stream()))

    @staticmethod
    def warp_bwd(in_, channels, d, field, gout, gin, gfield):
        _check(_capi.lib().mdg_warp_bwd(_ptr(in_), channels, dims3(d), _ptr(field), _ptr(gout),
                                        _ptr(gin), _ptr(gfield), _stream()))

    @staticmethod
    def upsample2_fwd(in_, channels, d, td, scale, out):
        _check(_capi.lib().mdg_upsample2_fwd(_ptr(in_), channels, dims3(d), dims3(td),
                                             float(scale), _ptr(out), _stream()))

    @staticmethod
    def upsample2_bwd(channels, d, td, scale, gout, gin):
        _check(_capi.lib().mdg_upsample2_bwd(channels, dims3(d), dims3(td), float(scale),
                                             _ptr(gout), _ptr(gin), _stream()))

    @staticmethod
    def conv3_fwd(in_, ic, d, k, bias, oc, out):
        _check(_capi.lib().mdg_conv3_fwd(_ptr(in_), ic, dims3(d), _ptr(k), _ptr(bias), oc,
                                         _ptr(out), _stream()))

    @staticmethod
    def conv3_bwd(in_, ic, d, k, oc, gout, gin, gk, gbias):
        _check(_capi.lib().mdg_conv3_bwd(_ptr(in_), ic, dims3(d), _ptr(k), oc, _ptr(gout),
                                         _ptr(gin), _ptr(gk), _ptr(gbias), _stream()))


# ------------------------------------------------------------------ op tier
def _empty(*shape, like):
    return torch.empty(*shape, dtype=torch.float32, device=like.device)


def _zeros(*shape, like):
    return torch.zeros(*shape, dtype=torch.float32, device=like.device)


def set_deterministic(on=True):
    """Deterministic mode (mdg_set_deterministic): bit-identical results from
    run to run, the warp / compose input gradients gathered per target instead
    of scattered with float atomics.  Returns the previous setting."""
    return bool(_capi.lib().mdg_set_deterministic(1 if on else 0))


def deterministic():
    return bool(_capi.lib().mdg_get_deterministic())


def check_numeric(d):
    """Raise NumericError if a fused-tier kernel saw a non-finite logit
    (position decoded against dims d)."""
    _check(_capi.lib().mdg_check_numeric(dims3(d), _stream()))


def modet_fwd(Q, K, B, d, cfg: AttentionConfig, layout=MDG_QK_POSMAJOR, want_w=False,
              check=True):
    """Fused ModeT forward: (SF {3S,n}, LSE {S,n}[, W {S,n,27}]).

    Equals subfields_fwd(na_fused_fwd(Q,K,B)) of the reference
    (attention.hpp:83-123, 282-298)."""
    cfg.validate()
    n = voxel_count(d)
    S, hd = cfg.heads, cfg.head_dim
    if Q.numel() != n * S * hd or K.shape != Q.shape:
        raise InvalidInput("neighborhood_attention: Q/K layout inconsistent with config")
    if B.numel() != S * cfg.window():
        raise InvalidInput("neighborhood_attention: bias must be {S, n^3}")
    SF = _empty(3 * S, n, like=Q)
    LSE = _empty(S, n, like=Q)
    W = _empty(S, n, cfg.window(), like=Q) if want_w else None
    _check(_capi.lib().mdg_modet_fwd(_ptr(Q), _ptr(K), _ptr(B), dims3(d), S, hd,
                                     cfg.neighborhood, layout, _ptr(SF), _ptr(LSE), _ptr(W),
                                     _stream()))
    if check:
        check_numeric(d)
    return (SF, LSE, W) if want_w else (SF, LSE)


def modet_bwd(Q, K, B, SF, LSE, gSF, d, cfg: AttentionConfig, layout=MDG_QK_POSMAJOR,
              gQ=None, gK=None, gB=None, accumulate=True):
    """Fused ModeT backward; accumulates into (and returns) gQ, gK, gB.
    Fresh gradient buffers are produced without a read-modify-write."""
    if gQ is None and gK is None:
        gQ, gK, acc = torch.empty_like(Q), torch.empty_like(K), False
    else:
        acc = accumulate
        gQ = _zeros(*Q.shape, like=Q) if gQ is None else gQ
        gK = _zeros(*K.shape, like=K) if gK is None else gK
    gB = _zeros(*B.shape, like=B) if gB is None else gB
    _check(_capi.lib().mdg_modet_bwd(_ptr(Q), _ptr(K), _ptr(B), _ptr(SF), _ptr(LSE), _ptr(gSF),
                                     dims3(d), cfg.heads, cfg.head_dim, cfg.neighborhood, layout,
                                     _ptr(gQ), _ptr(gK), _ptr(gB), int(acc), _stream()))
    return gQ, gK, gB


def na_fused(Q, K, B, d, cfg: AttentionConfig):
    """op_na_fused forward value (attention.hpp:373-390): W {S, n, nb^3}."""
    cfg.validate()
    n = voxel_count(d)
    if Q.dim() != 2 or Q.shape[0] != n or Q.shape[1] != cfg.heads * cfg.head_dim or \
            K.shape != Q.shape:
        raise InvalidInput("neighborhood_attention: Q/K layout inconsistent with config")
    if B.numel() != cfg.heads * cfg.window():
        raise InvalidInput("neighborhood_attention: bias must be {S, n^3}")
    W = _empty(cfg.heads, n, cfg.window(), like=Q)
    kern.na_fused_fwd(Q, K, B, d, cfg.heads, cfg.head_dim, cfg.neighborhood, W)
    return W


def subfields(W, d, cfg: AttentionConfig, norm_tol=1e-5):
    """op_subfields forward value (attention.hpp:414-436) incl. the row check."""
    n = voxel_count(d)
    if W.dim() != 3 or W.shape[0] != cfg.heads or W.shape[1] != n or W.shape[2] != cfg.window():
        raise InvalidInput("subfields: weights must be {S, n, win}")
    _check(_capi.lib().mdg_subfields_check_rows(_ptr(W), dims3(d), cfg.heads, cfg.neighborhood,
                                                float(norm_tol), _stream()))
    out = _empty(3 * cfg.heads, n, like=W)
    kern.subfields_fwd(W, d, cfg.heads, cfg.neighborhood, out)
    return out


def warp(vol, field, d=None):
    """op_warp / field_ops warp forward: vol {C, l, w, h}, field {3, l, w, h}."""
    if d is None:
        d = (vol.shape[-1], vol.shape[-2], vol.shape[-3])
    Cc = vol.numel() // voxel_count(d)
    if field.numel() != 3 * voxel_count(d):
        raise InvalidInput(f"warp: field must be {{3,{d[0]}x{d[1]}x{d[2]}}}")
    out = torch.empty_like(vol)
    kern.warp_fwd(vol, Cc, d, field, out)
    return out


def warp_bwd(vol, field, gout, d=None, gin=None, gfield=None, want_gin=True, want_gfield=True):
    if d is None:
        d = (vol.shape[-1], vol.shape[-2], vol.shape[-3])
    Cc = vol.numel() // voxel_count(d)
    if want_gin and gin is None:
        gin = torch.zeros_like(vol)
    if want_gfield and gfield is None:
        gfield = torch.zeros_like(field)
    kern.warp_bwd(vol, Cc, d, field, gout, gin if want_gin else None,
                  gfield if want_gfield else None)
    return gin, gfield


def compose(prev, res, d=None):
    """compose(prev, res)(x) = res(x) + prev(x + res(x)) (field_ops.hpp:42-49)."""
    if prev.shape != res.shape:
        raise InvalidInput("compose: field dims mismatch")
    if d is None:
        d = (prev.shape[-1], prev.shape[-2], prev.shape[-3])
    out = torch.empty_like(prev)
    _check(_capi.lib().mdg_compose_fwd(_ptr(prev), _ptr(res), dims3(d), _ptr(out), _stream()))
    return out


def compose_bwd(prev, res, gout, d=None, gprev=None, gres=None):
    if d is None:
        d = (prev.shape[-1], prev.shape[-2], prev.shape[-3])
    gprev = torch.zeros_like(prev) if gprev is None else gprev
    gres = torch.zeros_like(res) if gres is None else gres
    _check(_capi.lib().mdg_compose_bwd(_ptr(prev), _ptr(res), dims3(d), _ptr(gout), _ptr(gprev),
                                       _ptr(gres), _stream()))
    return gprev, gres


def upsample_field_2x(field, target, d=None):
    """op_upsample_field_2x forward (ops.hpp:258-271): values x2 on the finer grid."""
    if d is None:
        d = (field.shape[-1], field.shape[-2], field.shape[-3])
    Cc = field.numel() // voxel_count(d)
    th, tw, tl = target
    out = _empty(Cc, tl, tw, th, like=field)
    kern.upsample2_fwd(field, Cc, d, target, 2.0, out)
    return out


def upsample_field_2x_bwd(gout, d, target, gin=None):
    Cc = gout.numel() // voxel_count(target)
    h, w, l = d
    gin = _zeros(Cc, l, w, h, like=gout) if gin is None else gin
    kern.upsample2_bwd(Cc, d, target, 2.0, gout, gin)
    return gin


def conv3(x, k, bias, d=None):
    """op_conv3 forward (ops.hpp:137-158); RegHead = conv3 with ic=3S, oc=3."""
    if d is None:
        d = (x.shape[-1], x.shape[-2], x.shape[-3])
    ic = x.numel() // voxel_count(d)
    if k.dim() != 5 or tuple(k.shape[2:]) != (3, 3, 3):
        raise InvalidInput("conv3: kernel must be {oc,ic,3,3,3}")
    if k.shape[1] != ic:
        raise InvalidInput("conv3: input channels do not match kernel")
    oc = k.shape[0]
    if bias is not None and bias.numel() != oc:
        raise InvalidInput("conv3: bias size mismatch")
    h, w, l = d
    out = _empty(oc, l, w, h, like=x)
    kern.conv3_fwd(x, ic, d, k, bias, oc, out)
    return out


def conv3_bwd(x, k, gout, d=None, gin=None, gk=None, gbias=None):
    if d is None:
        d = (x.shape[-1], x.shape[-2], x.shape[-3])
    ic = x.numel() // voxel_count(d)
    oc = k.shape[0]
    gin = torch.zeros_like(x) if gin is None else gin
    gk = torch.zeros_like(k) if gk is None else gk
    gbias = _zeros(oc, like=k) if gbias is None else gbias
    kern.conv3_bwd(x, ic, d, k, oc, gout, gin, gk, gbias)
    return gin, gk, gbias


def scaling_squaring(vel, steps, d=None, keep=False):
    """reghead.hpp:52-67.  keep=True also returns the saved intermediates."""
    if steps < 1:
        raise InvalidInput("scaling_squaring: steps must be >= 1")
    if d is None:
        d = (vel.shape[-1], vel.shape[-2], vel.shape[-3])
    out = torch.empty_like(vel)
    saved = _empty(steps + 1, *vel.shape, like=vel) if keep else None
    _check(_capi.lib().mdg_scaling_squaring_fwd(_ptr(vel), dims3(d), steps, _ptr(out),
                                                _ptr(saved), _stream()))
    return (out, saved) if keep else out


def scaling_squaring_bwd(saved, steps, gout, d=None, gvel=None):
    if d is None:
        d = (gout.shape[-1], gout.shape[-2], gout.shape[-3])
    gvel = torch.zeros_like(gout) if gvel is None else gvel
    _check(_capi.lib().mdg_scaling_squaring_bwd(_ptr(saved), dims3(d), steps, _ptr(gout),
                                                _ptr(gvel), _stream()))
    return gvel


def qk_posmajor_to_planar(x):
    n, Cc = x.shape
    out = torch.empty(Cc, n, dtype=x.dtype, device=x.device)
    _check(_capi.lib().mdg_qk_posmajor_to_planar(_ptr(x), n, Cc, _ptr(out), _stream()))
    return out


def qk_planar_to_posmajor(x):
    Cc, n = x.shape
    out = torch.empty(n, Cc, dtype=x.dtype, device=x.device)
    _check(_capi.lib().mdg_qk_planar_to_posmajor(_ptr(x), n, Cc, _ptr(out), _stream()))
    return out


@dataclass
class ProjectionParams:
    """attention.hpp:323-328 (weight {K, C}, bias / ln_gamma / ln_beta {K})."""

    weight: torch.Tensor
    bias: torch.Tensor
    ln_gamma: torch.Tensor
    ln_beta: torch.Tensor


def project_qk(f, m, p: ProjectionParams, layout=MDG_QK_POSMAJOR):
    """op_project_qk forward (attention.hpp:351-356): Q = LN(W F + b),
    K = LN(W M + b).  f, m {C, n...}; returns Q, K as {n, K} (posmajor) or
    {K, n} (planar)."""
    Cc = f.shape[0]
    n = f.numel() // Cc
    if m.shape != f.shape:
        raise InvalidInput("project_qk: shape mismatch")
    if p.weight.dim() != 2 or p.weight.shape[1] != Cc:
        raise InvalidInput("linear_proj: weight shape must be {K,c} with matching channels")
    Kd = p.weight.shape[0]
    if p.bias.numel() != Kd:
        raise InvalidInput("linear_proj: bias size mismatch")
    if p.ln_gamma.numel() != Kd or p.ln_beta.numel() != Kd:
        raise InvalidInput("layer_norm: affine size mismatch")
    shape = (n, Kd) if layout == MDG_QK_POSMAJOR else (Kd, n)
    Q, K = _empty(*shape, like=f), _empty(*shape, like=f)
    _check(_capi.lib().mdg_project_qk_fwd(_ptr(f), _ptr(m), Cc, n, _ptr(p.weight), _ptr(p.bias),
                                          _ptr(p.ln_gamma), _ptr(p.ln_beta), Kd, layout,
                                          _ptr(Q), _ptr(K), _stream()))
    return Q, K


def project_qk_bwd(f, m, p: ProjectionParams, gQ, gK, layout=MDG_QK_POSMAJOR, gf=None, gm=None,
                   grads: ProjectionParams | None = None):
    """Backward of op_project_qk; accumulates into (and returns) gf, gm and the
    parameter gradients (a ProjectionParams of gradient tensors)."""
    Cc = f.shape[0]
    n = f.numel() // Cc
    Kd = p.weight.shape[0]
    gf = torch.zeros_like(f) if gf is None else gf
    gm = torch.zeros_like(m) if gm is None else gm
    if grads is None:
        grads = ProjectionParams(torch.zeros_like(p.weight), torch.zeros_like(p.bias),
                                 torch.zeros_like(p.ln_gamma), torch.zeros_like(p.ln_beta))
    _check(_capi.lib().mdg_project_qk_bwd(
        _ptr(f), _ptr(m), Cc, n, _ptr(p.weight), _ptr(p.bias), _ptr(p.ln_gamma), Kd, layout,
        _ptr(gQ), _ptr(gK), _ptr(gf), _ptr(gm), _ptr(grads.weight), _ptr(grads.bias),
        _ptr(grads.ln_gamma), _ptr(grads.ln_beta), _stream()))
    return gf, gm, grads


@dataclass
class LevelParams:
    """engine.hpp:108-112 LevelParams (projection, rel_pos_bias {S, 27},
    RegHead weight {3, 3S, 3, 3, 3} and bias {3})."""

    proj: ProjectionParams
    rel_pos_bias: torch.Tensor
    rh_weight: torch.Tensor
    rh_bias: torch.Tensor

    def tensors(self):
        """ModelParams::all_tensors order (engine.hpp:127-131)."""
        return [self.proj.weight, self.proj.bias, self.proj.ln_gamma, self.proj.ln_beta,
                self.rel_pos_bias, self.rh_weight, self.rh_bias]

    @staticmethod
    def from_tensors(ts):
        return LevelParams(ProjectionParams(*ts[:4]), ts[4], ts[5], ts[6])

    def zeros_like(self):
        return LevelParams.from_tensors([torch.zeros_like(t) for t in self.tensors()])


@dataclass
class LossConfig:
    """objective.hpp:21-31 (lambda, NCC window)."""

    lam: float = 1.0
    ncc_window: int = 9


def total_loss(fixed, moving, phi, cfg: LossConfig = LossConfig(), want_warped=False):
    """op_total_loss forward (objective.hpp:71-78).  fixed / moving {1,l,w,h}
    (or {l,w,h}), phi {3,l,w,h}.  Returns a device tensor {total, ncc, reg}
    (and the warped moving image)."""
    l, w, h = phi.shape[-3:]
    if fixed.numel() != l * w * h or moving.shape != fixed.shape:
        raise InvalidInput("ncc_loss: expects single-channel volumes of the field's dims")
    terms = _empty(3, like=phi)
    warped = torch.empty_like(moving) if want_warped else None
    _check(_capi.lib().mdg_total_loss_fwd(_ptr(fixed), _ptr(moving), _ptr(phi),
                                          dims3((h, w, l)), cfg.ncc_window, float(cfg.lam),
                                          _ptr(terms), _ptr(warped), _stream()))
    return (terms, warped) if want_warped else terms


def total_loss_bwd(fixed, moving, phi, cfg: LossConfig = LossConfig(), seed=1.0, gphi=None,
                   gmoving=None):
    """Backward of seed * total: accumulates into (and returns) gphi, gmoving."""
    l, w, h = phi.shape[-3:]
    gphi = torch.zeros_like(phi) if gphi is None else gphi
    gmoving = torch.zeros_like(moving) if gmoving is None else gmoving
    _check(_capi.lib().mdg_total_loss_bwd(_ptr(fixed), _ptr(moving), _ptr(phi),
                                          dims3((h, w, l)), cfg.ncc_window, float(cfg.lam),
                                          float(seed), _ptr(gphi), _ptr(gmoving), _stream()))
    return gphi, gmoving


def _iptr(t, name="labels"):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.int32 \
            or not t.is_contiguous():
        raise InvalidInput(f"{name}: must be a contiguous CUDA int32 tensor")
    return t.data_ptr()


def warp_labels(labels, phi):
    """metrics.cpp:145-164: nearest-neighbour warp of an int32 label volume
    {l,w,h} (or {1,l,w,h}) by phi {3,l,w,h} (bit-identical)."""
    l, w, h = phi.shape[-3:]
    if labels.numel() != l * w * h:
        raise InvalidInput("warp_labels: dims mismatch")
    out = torch.empty_like(labels)
    _check(_capi.lib().mdg_warp_labels(_iptr(labels), dims3((h, w, l)), _ptr(phi),
                                       _iptr(out, "out"), _stream()))
    return out


def mean_dice(a, b, max_label=None):
    """metrics.cpp:100-129 mean Dice over the labels present (0 excluded);
    returns a Python float (bit-identical to the reference's double)."""
    if a.shape != b.shape:
        raise InvalidInput("dice: dims mismatch")
    if max_label is None:
        max_label = int(torch.maximum(a.max(), b.max()).item()) if a.numel() else 0
    out = C.c_double()
    _check(_capi.lib().mdg_mean_dice(_iptr(a, "a"), _iptr(b, "b"), a.numel(), int(max_label),
                                     C.byref(out), _stream()))
    return out.value


class AdamOptimizer:
    """engine.hpp:268-304 AdamOptimizer over a list of CUDA parameter tensors;
    step(lr, grads) updates them in place (bit-identical double arithmetic)."""

    def __init__(self, params, beta1=0.9, beta2=0.999, eps=1e-8):
        self.params = list(params)
        self.m = [torch.zeros_like(p) for p in self.params]
        self.v = [torch.zeros_like(p) for p in self.params]
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.t = 0

    def step(self, lr, grads):
        self.t += 1
        L = _capi.lib()
        for p, g, m, v in zip(self.params, grads, self.m, self.v):
            _check(L.mdg_adam_step(_ptr(p), _ptr(g), _ptr(m), _ptr(v), p.numel(), float(lr),
                                   self.beta1, self.beta2, self.eps, self.t, _stream()))


def sgd_step(params, grads, lr):
    """engine.hpp:306-311."""
    for p, g in zip(params, grads):
        _check(_capi.lib().mdg_sgd_step(_ptr(p), _ptr(g), p.numel(), float(lr), _stream()))


@dataclass
class ModelConfig:
    """engine.hpp:30-78 (decoder part): heads coarse -> fine, head_dim,
    neighborhood, diffeomorphic + ss_steps."""

    heads_per_level: tuple = (8, 4, 2, 1, 1)
    head_dim: int = 6
    neighborhood: int = 3
    diffeomorphic: bool = False
    ss_steps: int = 7


class Pyramid:
    """The decoding pyramid (build_pipeline engine.hpp:179-219 minus the encoder)
    on device-resident features, driven by libmdg's native driver.

    ``dims`` / ``channels``: level grids and feature channels, coarse -> fine."""

    def __init__(self, cfg: ModelConfig, dims, channels, check_finite=True):
        L = len(dims)
        if len(cfg.heads_per_level) != L or len(channels) != L:
            raise InvalidInput("model: heads_per_level must have one entry per level")
        if L > _capi.MAX_LEVELS:
            raise InvalidInput("pyramid: too many levels")
        c = _capi.PyramidConfig()
        c.levels = L
        for k in range(L):
            c.heads[k] = int(cfg.heads_per_level[k])
            c.channels[k] = int(channels[k])
            c.dims[k] = dims3(dims[k])
        c.head_dim, c.neighborhood = cfg.head_dim, cfg.neighborhood
        c.diffeomorphic, c.ss_steps = int(cfg.diffeomorphic), cfg.ss_steps
        c.check_finite = int(check_finite)
        self.cfg, self.dims, self.channels = cfg, [tuple(d) for d in dims], list(channels)
        self._L = _capi.lib()
        h = C.c_void_p()
        _check(self._L.mdg_pyramid_create(C.byref(c), C.byref(h)))
        self._h = h
        self._keep = None

    def __del__(self):
        try:
            if self._h:
                self._L.mdg_pyramid_destroy(self._h)
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        return int(self._L.mdg_pyramid_bytes(self._h))

    @staticmethod
    def _ptrs(ts):
        arr = (C.c_void_p * len(ts))()
        for i, t in enumerate(ts):
            arr[i] = _ptr(t) if t is not None else None
        return arr

    @staticmethod
    def _level_structs(levels, cls):
        arr = (cls * len(levels))()
        for i, lp in enumerate(levels):
            for f, t in zip(_capi.LEVEL_FIELDS, lp.tensors()):
                setattr(arr[i], f, _ptr(t) if t is not None else None)
        return arr

    def forward(self, f_feats, m_feats, params, want_residuals=False):
        """Returns phi {3, fine dims} (and the per-level residuals)."""
        L = len(self.dims)
        fine = self.dims[-1]
        phi = torch.empty(3, fine[2], fine[1], fine[0], dtype=torch.float32,
                          device=f_feats[-1].device)
        res = [torch.empty(3, d[2], d[1], d[0], dtype=torch.float32, device=phi.device)
               for d in self.dims] if want_residuals else None
        for k in range(L):
            n = voxel_count(self.dims[k])
            if f_feats[k].numel() != self.channels[k] * n or m_feats[k].shape != f_feats[k].shape:
                raise InvalidInput(f"pyramid: level {k} feature shape mismatch")
        fp, mp = self._ptrs(f_feats), self._ptrs(m_feats)
        ps = self._level_structs(params, _capi.LevelParams)
        rp = self._ptrs(res) if res is not None else None
        self._keep = (list(f_feats), list(m_feats), list(params))  # saved for backward
        _check(self._L.mdg_pyramid_forward(self._h, fp, mp, ps, _ptr(phi), rp, _stream()))
        return (phi, res) if want_residuals else phi

    def backward(self, gphi, grads=None, gf=None, gm=None):
        """Accumulates into grads (list of LevelParams of gradient tensors) and the
        feature gradients gf / gm (lists); returns (grads, gf, gm)."""
        if self._keep is None:
            raise InvalidInput("pyramid: backward without a forward")
        f_feats, m_feats, params = self._keep
        grads = [p.zeros_like() for p in params] if grads is None else grads
        gf = [torch.zeros_like(t) for t in f_feats] if gf is None else gf
        gm = [torch.zeros_like(t) for t in m_feats] if gm is None else gm
        gs = self._level_structs(grads, _capi.LevelGrads)
        _check(self._L.mdg_pyramid_backward(self._h, _ptr(gphi), gs, self._ptrs(gf),
                                            self._ptrs(gm), _stream()))
        return grads, gf, gm


@dataclass
class BlockParams:
    """encoder.hpp:45-48 ConvBlockParams: w1 {C,Cin,3,3,3}, b1/g1/be1 {C},
    w2 {C,C,3,3,3}, b2/g2/be2 {C}."""

    w1: torch.Tensor
    b1: torch.Tensor
    g1: torch.Tensor
    be1: torch.Tensor
    w2: torch.Tensor
    b2: torch.Tensor
    g2: torch.Tensor
    be2: torch.Tensor

    def tensors(self):
        return [self.w1, self.b1, self.g1, self.be1, self.w2, self.b2, self.g2, self.be2]

    def zeros_like(self):
        return BlockParams(*[torch.zeros_like(t) for t in self.tensors()])


class Encoder:
    """op_encode (encoder.hpp:102-116) on one image at a time; the object owns
    the saved activations of its last forward (one per image of a pair)."""

    def __init__(self, dims, base_channels=8, levels=5, slope=0.2):
        self._L = _capi.lib()
        h = C.c_void_p()
        _check(self._L.mdg_encoder_create(dims3(dims), base_channels, levels, float(slope),
                                          C.byref(h)))
        self._h = h
        self.dims = [tuple(int(v) for v in dims)]
        for _ in range(levels - 1):
            self.dims.append(halved(self.dims[-1]))
        self.channels = [base_channels << k for k in range(levels)]

    def __del__(self):
        try:
            if self._h:
                self._L.mdg_encoder_destroy(self._h)
        except Exception:
            pass

    def forward(self, image, blocks):
        feats = [torch.empty(c, d[2], d[1], d[0], dtype=torch.float32, device=image.device)
                 for c, d in zip(self.channels, self.dims)]
        bp = (_capi.BlockParams * len(blocks))()
        for i, b in enumerate(blocks):
            for f, t in zip(_capi.BLOCK_FIELDS, b.tensors()):
                setattr(bp[i], f, _ptr(t))
        fp = (C.c_void_p * len(feats))(*[_ptr(t) for t in feats])
        self._keep = (image, list(blocks))  # the backward reads the image and weights
        _check(self._L.mdg_encoder_forward(self._h, _ptr(image), bp, fp, _stream()))
        return feats

    def backward(self, gfeats, grads, gimage=None):
        gp = (C.c_void_p * len(gfeats))(*[_ptr(t) if t is not None else None for t in gfeats])
        gb = (_capi.BlockGrads * len(grads))()
        for i, g in enumerate(grads):
            for f, t in zip(_capi.BLOCK_FIELDS, g.tensors()):
                setattr(gb[i], f, _ptr(t))
        _check(self._L.mdg_encoder_backward(self._h, gp, gb, _ptr(gimage), _stream()))


def init_model(seed=42, base_channels=8, heads=(8, 4, 2, 1, 1), head_dim=6):
    """init_model(ModelConfig::small_preset(), seed) (engine.hpp:143-166): the
    75 parameter tensors in ModelParams::all_tensors order, drawn from the
    reference's Rng stream in the reference's order (bit-identical values).
    Host (CPU) tensors; move them to the device for ops.Model."""
    r = Rng(seed)
    out = []

    def kaiming(oc, ic):  # make_conv_block (encoder.hpp:52-57)
        bound = (6.0 / (ic * 27.0)) ** 0.5
        return r.uniform((oc, ic, 3, 3, 3), -bound, bound)

    for k in range(5):
        c = base_channels << k
        cin = 1 if k == 0 else base_channels << (k - 1)
        w1 = kaiming(c, cin)
        w2 = kaiming(c, c)
        out += [w1, torch.zeros(c), torch.ones(c), torch.zeros(c),
                w2, torch.zeros(c), torch.ones(c), torch.zeros(c)]
    for k in range(5):
        cin = base_channels << (4 - k)
        S = heads[k]
        K = S * head_dim
        pw = r.normal((K, cin), 0.0, 1e-5)          # make_projection_params
        rh = r.normal((3, 3 * S, 3, 3, 3), 0.0, 1e-5)  # make_reghead_params
        out += [pw, torch.zeros(K), torch.ones(K), torch.zeros(K), torch.zeros(S, 27), rh,
                torch.zeros(3)]
    return out


class Model:
    """ModelParams (engine.hpp:114-140) of the small preset as device tensors,
    in the ModelParams::all_tensors order (5 encoder blocks, then 5 decoder
    levels coarse -> fine), plus one pairwise-optimisation step
    (run_loss_step engine.hpp:316-340 + an Adam update)."""

    def __init__(self, tensors, dims, cfg: ModelConfig = None, loss: LossConfig = None,
                 base_channels=8):
        self.cfg = cfg or ModelConfig()
        self.loss_cfg = loss or LossConfig()
        self.tensors = list(tensors)
        assert len(self.tensors) == 75, "expects the 75 ModelParams tensors"
        self.blocks = [BlockParams(*self.tensors[8 * k:8 * k + 8]) for k in range(5)]
        self.levels = [LevelParams.from_tensors(self.tensors[40 + 7 * k:47 + 7 * k])
                       for k in range(5)]
        self.enc_f = Encoder(dims, base_channels)
        self.enc_m = Encoder(dims, base_channels)
        pdims = self.enc_f.dims[::-1]
        pch = self.enc_f.channels[::-1]
        self.pyr = Pyramid(self.cfg, pdims, pch)
        self.grads = [torch.zeros_like(t) for t in self.tensors]
        self.opt = AdamOptimizer(self.tensors)

    def _grad_structs(self):
        gb = [BlockParams(*self.grads[8 * k:8 * k + 8]) for k in range(5)]
        gl = [LevelParams.from_tensors(self.grads[40 + 7 * k:47 + 7 * k]) for k in range(5)]
        return gb, gl

    def loss_step(self, fixed, moving, backward=True):
        """Forward (encoder x2 -> pyramid -> loss) and, optionally, the backward
        into self.grads (zeroed first).  Returns (terms {total,ncc,reg}, phi)."""
        ff = self.enc_f.forward(fixed, self.blocks)
        mf = self.enc_m.forward(moving, self.blocks)
        phi = self.pyr.forward(ff[::-1], mf[::-1], self.levels)
        terms = total_loss(fixed, moving, phi, self.loss_cfg)
        if backward:
            for g in self.grads:
                g.zero_()
            gphi = total_loss_bwd(fixed, moving, phi, self.loss_cfg)[0]
            gb, gl = self._grad_structs()
            gf = [torch.zeros_like(t) for t in ff[::-1]]
            gm = [torch.zeros_like(t) for t in mf[::-1]]
            self.pyr.backward(gphi, gl, gf, gm)
            self.enc_f.backward(gf[::-1], gb)
            self.enc_m.backward(gm[::-1], gb)
        return terms, phi

    def po_step(self, fixed, moving, lr=1e-4):
        """One PO iteration (engine.hpp:389-398): loss + backward + Adam."""
        terms, phi = self.loss_step(fixed, moving, backward=True)
        self.opt.step(lr, self.grads)
        return terms, phi

    def pairwise_optimize(self, fixed, moving, iters=50, lr=1e-4, labels_fixed=None,
                          labels_moving=None):
        """pairwise_optimize (engine.hpp:377-411): `iters` updates then a final
        evaluation; returns (loss_trace, dice_trace, phi) like PoResult."""
        loss_trace, dice_trace = [], []
        with_dice = labels_fixed is not None and labels_moving is not None
        phi = None
        for i in range(iters + 1):
            last = i == iters
            terms, phi = self.loss_step(fixed, moving, backward=not last)
            loss = float(terms[0])  # synchronises: the reference checks the loss
            if not (loss == loss and abs(loss) != float("inf")):
                raise NumericError(f"optimization: non-finite loss ({loss})")
            loss_trace.append(loss)
            if with_dice:
                dice_trace.append(mean_dice(labels_fixed, warp_labels(labels_moving, phi)))
            if not last:
                self.opt.step(lr, self.grads)
        return loss_trace, dice_trace, phi


def init_model_cfg(config, seed=42):
    """init_model(cfg, seed) (engine.hpp:143-166) for any model_config(...) by
    libmdg on the host: the ModelParams::all_tensors list (CPU tensors),
    bit-identical to the reference."""
    L = _capi.lib()
    nt = C.c_int()
    sizes = (C.c_int64 * 128)()
    L.mdg_config_param_count(C.byref(config), C.byref(nt), sizes)
    out = [torch.empty(int(sizes[i]), dtype=torch.float32) for i in range(nt.value)]
    ptrs = (C.c_void_p * nt.value)(*[t.data_ptr() for t in out])
    _check(L.mdg_model_init_cfg(C.byref(config), seed, ptrs))
    return out


def init_model_native(seed=42):
    """mdg_model_init: init_model(small_preset, seed) drawn by libmdg on the
    host (no device needed); the same 75 tensors as init_model()."""
    L = _capi.lib()
    nt = C.c_int(0)
    L.mdg_model_param_count(C.byref(nt), None)
    sizes = (C.c_int64 * nt.value)()
    L.mdg_model_param_count(None, sizes)
    shapes = [t.shape for t in _preset_meta()]
    out = [torch.empty(int(s), dtype=torch.float32) for s in sizes]
    ptrs = (C.c_void_p * nt.value)(*[t.data_ptr() for t in out])
    _check(L.mdg_model_init(seed, ptrs))
    return [t.view(s) for t, s in zip(out, shapes)]


def _preset_meta(base_channels=8, heads=(8, 4, 2, 1, 1), head_dim=6):
    out = []
    for k in range(5):
        c = base_channels << k
        cin = 1 if k == 0 else base_channels << (k - 1)
        out += [torch.empty(c, cin, 3, 3, 3, device="meta")] + \
               [torch.empty(c, device="meta")] * 3 + \
               [torch.empty(c, c, 3, 3, 3, device="meta")] + [torch.empty(c, device="meta")] * 3
    for k in range(5):
        cin, S = base_channels << (4 - k), heads[k]
        K = S * head_dim
        out += [torch.empty(K, cin, device="meta")] + [torch.empty(K, device="meta")] * 3 + \
               [torch.empty(S, 27, device="meta"), torch.empty(3, 3 * S, 3, 3, 3, device="meta"),
                torch.empty(3, device="meta")]
    return out


class NativeModel:
    """The whole model as libmdg's native object (mdg_model_*): encoder x2 ->
    pyramid -> loss -> backward -> Adam composed in C++ with no framework
    underneath.  Same contract as Model; `tensors` are the 75 device
    parameters (updated in place by po_step)."""

    def __init__(self, tensors, dims, loss: LossConfig = None, check_finite=False, config=None,
                 optimizer="adam"):
        """config: a model_config(...) (default: the small preset);
        optimizer: "adam" (AdamOptimizer) or "sgd" (sgd_step), engine.hpp:80."""
        self._L = _capi.lib()
        self.tensors = list(tensors)
        self.config = config if config is not None else model_config()
        if optimizer not in ("adam", "sgd"):
            raise InvalidInput("model: optimizer must be 'adam' or 'sgd'")
        nt = C.c_int()
        sizes = (C.c_int64 * 128)()
        self._L.mdg_config_param_count(C.byref(self.config), C.byref(nt), sizes)
        if len(self.tensors) != nt.value:
            raise InvalidInput(f"model: expects the {nt.value} ModelParams tensors")
        for i, t in enumerate(self.tensors):
            _ptr(t, f"model tensor {i}")
            if t.numel() != sizes[i]:
                raise InvalidInput(f"model: tensor {i} has {t.numel()} elements, the model "
                                   f"expects {sizes[i]}")
        self.dims = tuple(int(v) for v in dims)
        lc = loss or LossConfig()
        ptrs = (C.c_void_p * len(self.tensors))(*[_ptr(t) for t in self.tensors])
        h = C.c_void_p()
        _check(self._L.mdg_model_create_cfg(C.byref(self.config), dims3(dims), ptrs,
                                            float(lc.lam), int(lc.ncc_window),
                                            1 if check_finite else 0,
                                            0 if optimizer == "adam" else 1, C.byref(h)))
        self._h = h
        n = voxel_count(self.dims)
        dev = self.tensors[0].device
        self._terms = torch.empty(3, device=dev)
        self._phi = torch.empty(3, *self.dims[::-1], device=dev)
        self.n = n

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.mdg_model_destroy(h)
            self._h = None

    @property
    def grads(self):
        g = self._L.mdg_model_grads(self._h)
        out = []
        for i, t in enumerate(self.tensors):
            ptr = g[i]
            out.append(_wrap_device(ptr, t.shape, t.device))
        return out

    def _check_images(self, fixed, moving):
        for name, t in (("fixed", fixed), ("moving", moving)):
            if t.numel() != self.n:
                raise InvalidInput(f"model: {name} image has {t.numel()} voxels, the model "
                                   f"was created for {self.n}")

    def loss_step(self, fixed, moving, backward=True):
        self._check_images(fixed, moving)
        _check(self._L.mdg_model_loss_step(self._h, _ptr(fixed, "fixed"), _ptr(moving, "moving"),
                                           1 if backward else 0, _ptr(self._terms),
                                           _ptr(self._phi), _stream()))
        return self._terms.clone(), self._phi.clone()

    def po_step(self, fixed, moving, lr=1e-4, graph=True):
        """loss + backward + the optimizer update; graph=True replays the
        iteration as one CUDA graph (mdg_model_po_step).  Returns (terms, phi)."""
        self._check_images(fixed, moving)
        if not graph:
            terms, phi = self.loss_step(fixed, moving, backward=True)
            _check(self._L.mdg_model_adam_step(self._h, float(lr), _stream()))
            return terms, phi
        _check(self._L.mdg_model_po_step(self._h, _ptr(fixed, "fixed"), _ptr(moving, "moving"),
                                         float(lr), _ptr(self._terms), _stream()))
        phi = _wrap_device(self._L.mdg_model_phi(self._h), self._phi.shape, self._phi.device)
        return self._terms.clone(), phi.clone()

    def pairwise_optimize(self, fixed, moving, iters=50, lr=1e-4, labels_fixed=None,
                          labels_moving=None, graph=True):
        """pairwise_optimize (engine.hpp:377-411) on the native driver: `iters`
        Adam updates (each one CUDA graph replay) then a final evaluation
        forward.  Returns (loss_trace, dice_trace, phi) like PoResult; the loss
        is read back and checked finite every iteration as the reference does."""
        loss_trace, dice_trace = [], []
        with_dice = labels_fixed is not None and labels_moving is not None
        phi = None
        for i in range(iters + 1):
            last = i == iters
            if last:
                terms, phi = self.loss_step(fixed, moving, backward=False)
            else:  # the returned loss/phi are the forward before this update
                terms, phi = self.po_step(fixed, moving, lr, graph=graph)
            loss = float(terms[0])
            if not (loss == loss and abs(loss) != float("inf")):
                raise NumericError(f"optimization: non-finite loss ({loss})")
            loss_trace.append(loss)
            if with_dice:
                dice_trace.append(mean_dice(labels_fixed, warp_labels(labels_moving, phi)))
        return loss_trace, dice_trace, phi


def _wrap_device(ptr, shape, device):
    """A torch view of libmdg-owned device memory (float32, contiguous); valid
    while the owning object lives."""
    n = 1
    for s in shape:
        n *= int(s)

    class _A:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_A(), device=device).view(shape)


def launch_count() -> int:
    return int(_capi.lib().mdg_launch_count())


class Rng:
    """Synthetic input stream bit-identical to mdreg::Rng (rng.hpp:23-67)."""

    def __init__(self, seed: int):
        self._L = _capi.lib()
        self._h = self._L.mdg_rng_new(seed)

    def __del__(self):
        try:
            self._L.mdg_rng_free(self._h)
        except Exception:
            pass

    def uniform(self, shape, lo=0.0, hi=1.0, out=None):
        out = torch.empty(shape, dtype=torch.float32) if out is None else out
        self._L.mdg_rng_fill_uniform(self._h, out.data_ptr(), out.numel(), lo, hi)
        return out

    def normal(self, shape, mean=0.0, sd=1.0, out=None):
        out = torch.empty(shape, dtype=torch.float32) if out is None else out
        self._L.mdg_rng_fill_normal(self._h, out.data_ptr(), out.numel(), mean, sd)
        return out


# ---------------------------------------------------------- synthetic inputs
def make_smooth_velocity(dims, seed, magnitude, sigma):
    """make_smooth_velocity (synth.cpp:75-90) on the host: {3, l, w, h} float32
    CPU tensor, bit-identical to the reference."""
    h, w, l = dims
    out = torch.empty(3, l, w, h, dtype=torch.float32)
    _check(_capi.lib().mdg_synth_smooth_velocity(dims3(dims), seed, magnitude, sigma,
                                                 out.data_ptr()))
    return out


def random_field(dims, seed, mag):
    """test::random_field (tests/test_util.hpp:40-48): i.i.d. displacement
    entries, the warp's worst case for gather locality.  {3, l, w, h} CPU."""
    h, w, l = dims
    out = torch.empty(3, l, w, h, dtype=torch.float32)
    _check(_capi.lib().mdg_synth_random_field(dims3(dims), seed, mag, out.data_ptr()))
    return out


def synth_pair(dims, seed=1, max_disp=2.0):
    """make_synth_pair (synth.cpp:92-192, SynthConfig defaults otherwise):
    (fixed {1,l,w,h}, moving, labels_fixed {l,w,h} int32, labels_moving, gt
    {3,l,w,h}) as CPU tensors.  Needs the device (the ground truth's
    scaling-and-squaring and the warps run there, bit-exact)."""
    h, w, l = dims
    f = torch.empty(1, l, w, h, dtype=torch.float32)
    m = torch.empty_like(f)
    lf = torch.empty(l, w, h, dtype=torch.int32)
    lm = torch.empty_like(lf)
    gt = torch.empty(3, l, w, h, dtype=torch.float32)
    _check(_capi.lib().mdg_synth_pair(dims3(dims), seed, max_disp, f.data_ptr(), m.data_ptr(),
                                      lf.data_ptr(), lm.data_ptr(), gt.data_ptr()))
    return f, m, lf, lm, gt


# ------------------------------------------------------------- file formats
# The reference's raw volume + JSON sidecar (io_raw.cpp) and MDT2 checkpoint
# (checkpoint.cpp) through libmdg's native readers / writers: host numpy
# arrays in the reference layouts ({l, w, h} volumes, {3, l, w, h} fields).
def _raw_load(fn, path, dtype, channels):
    import numpy as np

    L = _capi.lib()
    h = _capi.RawHeader()
    _check(getattr(L, fn)(str(path).encode(), C.byref(h), None))
    d = h.dims
    shape = ((channels,) if channels > 1 else ()) + (d.l, d.w, d.h)
    out = np.empty(shape, dtype=dtype)
    _check(getattr(L, fn)(str(path).encode(), C.byref(h), out.ctypes.data_as(C.c_void_p)))
    return out, tuple(float(v) for v in h.spacing)


def load_raw_volume(json_path):
    """load_raw_volume (io_raw.cpp:142-152) -> (f32 {l,w,h}, spacing)."""
    import numpy as np

    return _raw_load("mdg_raw_load_volume", json_path, np.float32, 1)


def load_raw_field(json_path):
    """load_raw_field (io_raw.cpp:160-169) -> f32 {3,l,w,h}."""
    import numpy as np

    return _raw_load("mdg_raw_load_field", json_path, np.float32, 3)[0]


def load_raw_labels(json_path):
    """load_raw_labels (io_raw.cpp:154-158) -> (int32 {l,w,h}, spacing)."""
    import numpy as np

    return _raw_load("mdg_raw_load_labels", json_path, np.int32, 1)


def load_nifti(path):
    """load_nifti (nifti.cpp:36-105) -> (f32 {l,w,h}, spacing)."""
    import numpy as np

    return _raw_load("mdg_nifti_load", path, np.float32, 1)


def _dims_of(a, channels):
    if a.ndim != 3 + (1 if channels > 1 else 0):
        raise InvalidInput("raw: array rank does not match")
    ll, w, h = a.shape[-3:]
    return Dims3(h, w, ll)


def save_raw_volume(base, vol, spacing=(1.0, 1.0, 1.0)):
    import numpy as np

    a = np.ascontiguousarray(vol, dtype=np.float32)
    sp = (C.c_float * 3)(*spacing)
    _check(_capi.lib().mdg_raw_save_volume(str(base).encode(), _dims_of(a, 1), sp,
                                           a.ctypes.data_as(C.c_void_p)))


def save_raw_field(base, field):
    import numpy as np

    a = np.ascontiguousarray(field, dtype=np.float32)
    _check(_capi.lib().mdg_raw_save_field(str(base).encode(), _dims_of(a, 3),
                                          a.ctypes.data_as(C.c_void_p)))


def save_raw_labels(base, labels, spacing=(1.0, 1.0, 1.0)):
    import numpy as np

    a = np.ascontiguousarray(labels, dtype=np.int32)
    sp = (C.c_float * 3)(*spacing)
    _check(_capi.lib().mdg_raw_save_labels(str(base).encode(), _dims_of(a, 1), sp,
                                           a.ctypes.data_as(C.c_void_p)))


def model_config(base_channels=8, leaky_slope=0.2, heads_per_level=(8, 4, 2, 1, 1), head_dim=6,
                 neighborhood=3, diffeomorphic=False, ss_steps=7):
    """A checkpoint ModelConfig (defaults: small_preset, engine.hpp:38-44)."""
    c = _capi.ModelConfigC()
    c.base_channels, c.leaky_slope = int(base_channels), float(leaky_slope)
    for i, v in enumerate(heads_per_level):
        c.heads_per_level[i] = int(v)
    c.head_dim, c.neighborhood = int(head_dim), int(neighborhood)
    c.diffeomorphic, c.ss_steps = 1 if diffeomorphic else 0, int(ss_steps)
    return c


def config_tensors(cfg):
    """(names, sizes) of ModelParams::all_tensors for a config."""
    L = _capi.lib()
    nt = C.c_int(0)
    L.mdg_config_param_count(C.byref(cfg), C.byref(nt), None)
    sizes = (C.c_int64 * nt.value)()
    L.mdg_config_param_count(C.byref(cfg), None, sizes)
    names = []
    buf = C.create_string_buffer(128)
    for i in range(nt.value):
        _check(L.mdg_config_tensor_name(C.byref(cfg), i, buf, 128))
        names.append(buf.value.decode())
    return names, [int(s) for s in sizes]


def save_checkpoint(path, tensors, cfg=None):
    """save_checkpoint (checkpoint.cpp:85-104): host float32 tensors in
    all_tensors order (numpy or CPU torch)."""
    import numpy as np

    cfg = cfg or model_config()
    arrs = [np.ascontiguousarray(np.asarray(t), dtype=np.float32) for t in tensors]
    names, sizes = config_tensors(cfg)
    if len(arrs) != len(sizes) or any(a.size != s for a, s in zip(arrs, sizes)):
        raise InvalidInput("checkpoint: tensors do not match the config's layout")
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    _check(_capi.lib().mdg_checkpoint_save(str(path).encode(), C.byref(cfg), ptrs))


def load_checkpoint(path):
    """load_checkpoint (checkpoint.cpp:106-145) -> (config, [float32 arrays],
    names)."""
    import numpy as np

    L = _capi.lib()
    cfg = _capi.ModelConfigC()
    _check(L.mdg_checkpoint_load(str(path).encode(), C.byref(cfg), None))
    names, sizes = config_tensors(cfg)
    arrs = [np.empty(s, dtype=np.float32) for s in sizes]
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    _check(L.mdg_checkpoint_load(str(path).encode(), C.byref(cfg), ptrs))
    return cfg, arrs, names
