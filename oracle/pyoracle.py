"""pyoracle — numpy/ctypes face of the CPU ORACLE.  TEST INFRASTRUCTURE ONLY.

Loads ``oracle/_build/libmdo.so`` (the C restatement, ``oracle/mdo.c``) and,
when present, ``oracle/_ref/libmdreg_ref.so`` (the unmodified reference headers
compiled by ``oracle/Makefile``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg import this module; the product package
never does.

Every wrapper takes/returns numpy float32 arrays in the reference layouts
(channel-major fields ``{C, l, w, h}`` in numpy index order, i.e. x fastest;
attention Q/K position-major ``{n, S*d}``; W ``{S, n, nb^3}``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_MDO = os.path.join(HERE, "_build", "libmdo.so")
LIB_REF = os.path.join(HERE, "_ref", "libmdreg_ref.so")

_f = C.POINTER(C.c_float)
_i = C.POINTER(C.c_int)


def build(quiet: bool = True) -> None:
    """Compile the restatement (and _ref when /root/reference is present)."""
    cmd = ["make", "-C", HERE, "-s"] if quiet else ["make", "-C", HERE]
    subprocess.run(cmd, check=True)


def _fp(a):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(_f)


class _Lib:
    """Common signatures for libmdo (prefix mdo_) and libmdreg_ref (mdr_)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L = self.lib
        p = prefix

        def sig(name, res, *args):
            fn = getattr(L, p + name)
            fn.restype = res
            fn.argtypes = list(args)
            return fn

        ii = C.c_int
        self._window_offset = sig("window_offset", None, ii, ii, _i)
        if prefix == "mdo_":
            self._na_fwd = sig("na_fwd", ii, _f, _f, _f, ii, ii, ii, ii, ii, ii, _f, _i)
        else:
            self._na_fwd = sig("na_fwd", ii, _f, _f, _f, ii, ii, ii, ii, ii, ii, _f)
            self._na_naive_fwd = sig("na_naive_fwd", ii, _f, _f, _f, ii, ii, ii, ii, ii, ii, _f)
            self._last_error = sig("last_error", C.c_char_p)
            self._smooth_vel = sig("make_smooth_velocity", None, ii, ii, ii, C.c_uint64,
                                   C.c_float, C.c_float, _f)
            self._attn_bench = sig("attention_bench_fused_ms", C.c_double, ii, ii, ii, ii, ii,
                                   ii, C.c_uint64)
            self._synth = sig("make_synth_pair", None, ii, ii, ii, C.c_uint64, C.c_float, _f, _f,
                              _i, _i, _f)
            self._warp_labels = sig("warp_labels", None, _i, ii, ii, ii, _f, _i)
            self._mean_dice = sig("mean_dice", C.c_double, _i, _i, ii, ii, ii)
        self._na_bwd = sig("na_bwd", None, _f, _f, _f, ii, ii, ii, ii, ii, ii, _f, _f, _f, _f)
        self._sf_fwd = sig("subfields_fwd", None, _f, ii, ii, ii, ii, ii, _f)
        self._sf_bwd = sig("subfields_bwd", None, ii, ii, ii, ii, ii, _f, _f)
        self._resolve = sig("resolve_axis", None, C.c_float, ii, _i, _i, _f, _i)
        self._warp_fwd = sig("warp_fwd", None, _f, ii, ii, ii, ii, _f, _f)
        self._warp_bwd = sig("warp_bwd", None, _f, ii, ii, ii, ii, _f, _f, _f, _f)
        self._up_fwd = sig("upsample2_fwd", None, _f, ii, ii, ii, ii, ii, ii, ii, C.c_float, _f)
        self._up_bwd = sig("upsample2_bwd", None, ii, ii, ii, ii, ii, ii, ii, C.c_float, _f, _f)
        self._up_ok = sig("upsample_target_ok", ii, ii, ii, ii, ii, ii, ii)
        self._conv_fwd = sig("conv3_fwd", None, _f, ii, ii, ii, ii, _f, _f, ii, _f)
        self._conv_bwd = sig("conv3_bwd", None, _f, ii, ii, ii, ii, _f, ii, _f, _f, _f, _f)
        self._comp_fwd = sig("compose_fwd", None, _f, _f, ii, ii, ii, _f)
        self._comp_bwd = sig("compose_bwd", None, _f, _f, ii, ii, ii, _f, _f, _f)
        self._ss = sig("scaling_squaring", None, _f, ii, ii, ii, ii, _f)
        i64 = C.c_int64
        dd = C.c_double
        if prefix == "mdo_":
            self._adam = sig("adam_step", None, _f, _f, _f, _f, i64, dd, dd, dd, dd, i64)
            self._lin_fwd = sig("linear_proj_fwd", None, _f, ii, i64, _f, _f, ii, _f)
            self._lin_bwd = sig("linear_proj_bwd", None, _f, ii, i64, _f, ii, _f, _f, _f, _f)
            self._ln_fwd = sig("layer_norm_fwd", None, _f, i64, ii, _f, _f, C.c_float, _f)
            self._ln_bwd = sig("layer_norm_bwd", None, _f, i64, ii, _f, C.c_float, _f, _f, _f,
                               _f)
        else:
            self._pqk = sig("project_qk", ii, _f, _f, ii, ii, ii, ii, _f, _f, _f, _f, ii, _f, _f,
                            _f, _f, _f, _f, _f, _f, _f, _f)
            pp = C.POINTER(_f)
            self._decoder = sig("decoder", ii, ii, _i, _i, _i, ii, ii, ii, ii, pp, pp, pp, _f,
                                _f, pp, pp, pp, pp)
            self._perr = sig("pipeline_error", C.c_char_p)
            self._adam_steps = sig("adam_steps", ii, _f, _f, i64, ii, dd, dd, dd, dd, _f, _f)
            self._mcount = sig("model_param_count", i64, C.c_uint64)
            self._mparams = sig("model_params", ii, C.c_uint64, _f, C.POINTER(i64))
            pp = C.POINTER(_f)
            self._encode = sig("encode", ii, _f, ii, ii, ii, _f, pp, pp, _f, _f)
            self._loss_step = sig("loss_step", ii, _f, _f, ii, ii, ii, _f, C.c_float, ii,
                                  C.POINTER(dd), _f, _f)
            self._po = sig("pairwise_optimize", ii, _f, _f, _i, _i, ii, ii, ii, _f, ii, dd, dd,
                           ii, C.POINTER(dd), C.POINTER(dd), _f)
            self._tloss = sig("total_loss", ii, _f, _f, _f, ii, ii, ii, ii, C.c_float, _f, _f,
                              _f, _f)
            self._lpc = sig("level_param_count", i64, ii, ii, ii, ii)

    # -- Q/K projection (ops.hpp:387-497, attention.hpp:351-356) -----------
    def project_qk(self, f, m, weight, bias, ln_g, ln_b, gQ=None, gK=None):
        """Q, K position-major {n, K}; with gQ/gK also returns the gradients
        (gf, gm, gweight, gbias, gln_g, gln_b) of sum(Q*gQ) + sum(K*gK)."""
        Cc = f.shape[0]
        n = f.size // Cc
        Kd = weight.shape[0]
        grads = None
        if self.prefix == "mdo_":
            eps = C.c_float(1e-5)
            outs = []
            raws = []
            for x in (f, m):
                raw = np.zeros((n, Kd), np.float32)
                self._lin_fwd(_fp(x), Cc, n, _fp(weight), _fp(bias), Kd, _fp(raw))
                out = np.zeros((n, Kd), np.float32)
                self._ln_fwd(_fp(raw), n, Kd, _fp(ln_g), _fp(ln_b), eps, _fp(out))
                raws.append(raw)
                outs.append(out)
            if gQ is not None:
                grads = [np.zeros_like(f), np.zeros_like(m), np.zeros_like(weight),
                         np.zeros_like(bias), np.zeros_like(ln_g), np.zeros_like(ln_b)]
                # tape order: K's nodes were pushed last, so they replay first
                for x, raw, g, gx in ((m, raws[1], gK, grads[1]), (f, raws[0], gQ, grads[0])):
                    graw = np.zeros((n, Kd), np.float32)
                    self._ln_bwd(_fp(raw), n, Kd, _fp(ln_g), eps, _fp(g), _fp(graw),
                                 _fp(grads[4]), _fp(grads[5]))
                    self._lin_bwd(_fp(x), Cc, n, _fp(weight), Kd, _fp(graw), _fp(gx),
                                  _fp(grads[2]), _fp(grads[3]))
            return (outs[0], outs[1], grads) if gQ is not None else (outs[0], outs[1])
        l, w, h = f.shape[1:]
        Q = np.zeros((n, Kd), np.float32)
        K = np.zeros((n, Kd), np.float32)
        if gQ is not None:
            grads = [np.zeros_like(f), np.zeros_like(m), np.zeros_like(weight),
                     np.zeros_like(bias), np.zeros_like(ln_g), np.zeros_like(ln_b)]
        g = grads or [None] * 6
        rc = self._pqk(_fp(f), _fp(m), Cc, h, w, l, _fp(weight), _fp(bias), _fp(ln_g),
                       _fp(ln_b), Kd, _fp(Q), _fp(K), _fp(gQ), _fp(gK), *[_fp(x) for x in g])
        if rc:
            raise RuntimeError(self._perr().decode())
        return (Q, K, grads) if gQ is not None else (Q, K)

    def decoder(self, dims, channels, heads, hd, f_feats, m_feats, params, gphi=None,
                diffeomorphic=False, ss_steps=7, nb=3):
        """Reference decoding pyramid (engine.hpp:189-216) on given features,
        coarse -> fine.  params[k]: packed level block (ModelParams order).
        Returns phi, residuals and (with gphi) (gparams, gf, gm)."""
        assert self.prefix == "mdr_"
        L = len(dims)
        dims_c = (C.c_int * (3 * L))(*[int(v) for d in dims for v in d])
        ch_c = (C.c_int * L)(*channels)
        hd_c = (C.c_int * L)(*heads)
        P = C.POINTER(C.c_float)
        arr = lambda xs: (P * L)(*[_fp(x) for x in xs])  # noqa: E731
        fine = dims[-1]
        phi = np.zeros((3, fine[2], fine[1], fine[0]), np.float32)
        res = [np.zeros((3, d[2], d[1], d[0]), np.float32) for d in dims]
        gparams = gf = gm = None
        if gphi is not None:
            gparams = [np.zeros_like(p) for p in params]
            gf = [np.zeros_like(x) for x in f_feats]
            gm = [np.zeros_like(x) for x in m_feats]
        rc = self._decoder(L, dims_c, ch_c, hd_c, hd, nb, int(diffeomorphic), ss_steps,
                           arr(f_feats), arr(m_feats), arr(params), _fp(gphi), _fp(phi),
                           arr(res), arr(gparams) if gparams else None,
                           arr(gf) if gf else None, arr(gm) if gm else None)
        if rc:
            raise RuntimeError(self._perr().decode())
        return (phi, res, (gparams, gf, gm)) if gphi is not None else (phi, res)

    def total_loss(self, fixed, moving, phi, window=9, lam=1.0, grads=True):
        """Reference op_total_loss: ({total, ncc, reg}, warped, gphi, gmoving)."""
        l, w, h = phi.shape[1:]
        terms = np.zeros(3, np.float32)
        warped = np.zeros_like(moving)
        gphi = np.zeros_like(phi) if grads else None
        gm = np.zeros_like(moving) if grads else None
        rc = self._tloss(_fp(fixed), _fp(moving), _fp(phi), h, w, l, window, lam, _fp(terms),
                         _fp(warped), _fp(gphi), _fp(gm))
        if rc:
            raise RuntimeError(self._perr().decode())
        return terms, warped, gphi, gm

    def adam(self, value, grads, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        """AdamOptimizer (engine.hpp:268-298): len(grads) consecutive steps from
        zero moments; returns the updated parameter."""
        value = value.copy()
        n = value.size
        if self.prefix == "mdo_":
            m = np.zeros_like(value)
            v = np.zeros_like(value)
            for t, g in enumerate(grads, start=1):
                self._adam(_fp(value), _fp(np.ascontiguousarray(g)), _fp(m), _fp(v), n, lr,
                           beta1, beta2, eps, t)
            return value
        G = np.ascontiguousarray(np.stack(grads)).astype(np.float32)
        rc = self._adam_steps(_fp(value), _fp(G), n, len(grads), lr, beta1, beta2, eps, None,
                              None)
        if rc:
            raise RuntimeError(self._perr().decode())
        return value

    def synth_pair(self, dims, seed=1, max_disp=2.0):
        """synth.cpp make_synth_pair: (fixed, moving, labels_fixed, labels_moving, gt)."""
        h, w, l = dims
        f = np.zeros((1, l, w, h), np.float32)
        m = np.zeros_like(f)
        lf = np.zeros((l, w, h), np.int32)
        lm = np.zeros_like(lf)
        gt = np.zeros((3, l, w, h), np.float32)
        ip = lambda a: a.ctypes.data_as(_i)  # noqa: E731
        self._synth(h, w, l, seed, max_disp, _fp(f), _fp(m), ip(lf), ip(lm), _fp(gt))
        return f, m, lf, lm, gt

    def warp_labels(self, labels, phi):
        l, w, h = phi.shape[1:]
        out = np.zeros_like(labels)
        ip = lambda a: np.ascontiguousarray(a).ctypes.data_as(_i)  # noqa: E731
        self._warp_labels(ip(labels), h, w, l, _fp(phi), out.ctypes.data_as(_i))
        return out

    def mean_dice(self, a, b):
        l, w, h = a.shape[-3:]
        ip = lambda x: np.ascontiguousarray(x, np.int32).ctypes.data_as(_i)  # noqa: E731
        return float(self._mean_dice(ip(a), ip(b), h, w, l))

    def model_params(self, seed=42):
        """init_model(small_preset, seed): (packed values, per-tensor sizes)."""
        n = int(self._mcount(seed))
        out = np.zeros(n, np.float32)
        sizes = (C.c_int64 * 128)()
        cnt = self._mparams(seed, _fp(out), sizes)
        return out, [int(sizes[i]) for i in range(cnt)]

    def encode(self, image, packed, gfeat=None):
        """op_encode of one image {1,l,w,h}: features (fine -> coarse) and, with
        gfeat, (gpacked, gimage) of sum_L <feat_L, gfeat_L>."""
        l, w, h = image.shape[1:]
        dims = [(h, w, l)]
        for _ in range(4):
            dims.append(tuple((v + 1) // 2 for v in dims[-1]))
        feats = [np.zeros((8 << k, d[2], d[1], d[0]), np.float32) for k, d in enumerate(dims)]
        P = C.POINTER(C.c_float)
        fa = (P * 5)(*[_fp(f) for f in feats])
        ga = (P * 5)(*[_fp(g) for g in gfeat]) if gfeat is not None else None
        gp = np.zeros_like(packed) if gfeat is not None else None
        gi = np.zeros_like(image) if gfeat is not None else None
        rc = self._encode(_fp(image), h, w, l, _fp(packed), fa, ga, _fp(gp), _fp(gi))
        if rc:
            raise RuntimeError(self._perr().decode())
        return (feats, gp, gi) if gfeat is not None else feats

    def loss_step(self, fixed, moving, packed, lam=1.0, window=9, grads=True):
        """run_loss_step (engine.hpp:316-340): (loss, gpacked, phi)."""
        l, w, h = fixed.shape[1:]
        loss = C.c_double()
        gp = np.zeros_like(packed) if grads else None
        phi = np.zeros((3, l, w, h), np.float32)
        rc = self._loss_step(_fp(fixed), _fp(moving), h, w, l, _fp(packed), lam, window,
                             C.byref(loss), _fp(gp), _fp(phi))
        if rc:
            raise RuntimeError(self._perr().decode())
        return loss.value, gp, phi

    def pairwise_optimize(self, fixed, moving, lf, lm, packed, iters, lr=1e-4, lam=1.0,
                          window=9):
        """pairwise_optimize (engine.hpp:377-411): (loss_trace, dice_trace, phi)."""
        l, w, h = fixed.shape[1:]
        lt = (C.c_double * (iters + 1))()
        dt = (C.c_double * (iters + 1))()
        phi = np.zeros((3, l, w, h), np.float32)
        ip = lambda a: np.ascontiguousarray(a, np.int32).ctypes.data_as(_i)  # noqa: E731
        rc = self._po(_fp(fixed), _fp(moving), ip(lf), ip(lm), h, w, l, _fp(packed), iters, lr,
                      lam, window, lt, dt, _fp(phi))
        if rc:
            raise RuntimeError(self._perr().decode())
        return list(lt), list(dt), phi

    # -- any ModelConfig / optimizer (reference build only) -----------------
    @staticmethod
    def _cfg(base=8, heads=(8, 4, 2, 1, 1), hd=6, diffeomorphic=False, ss_steps=7):
        return (C.c_int * 9)(base, *heads, hd, 1 if diffeomorphic else 0, ss_steps)

    def model_params_cfg(self, seed=42, **cfg):
        """init_model(cfg, seed): (packed, sizes); cfg keys: base, heads, hd,
        diffeomorphic, ss_steps."""
        c = self._cfg(**cfg)
        f = self.lib.mdr_model_param_count_cfg
        f.restype, f.argtypes = C.c_int64, [C.POINTER(C.c_int)]
        n = int(f(c))
        g = self.lib.mdr_model_params_cfg
        g.restype = C.c_int
        g.argtypes = [C.POINTER(C.c_int), C.c_uint64, _f, C.POINTER(C.c_int64)]
        out = np.zeros(n, np.float32)
        sizes = (C.c_int64 * 128)()
        cnt = g(c, seed, _fp(out), sizes)
        return out, [int(sizes[i]) for i in range(cnt)]

    def loss_step_cfg(self, fixed, moving, packed, lam=1.0, window=9, grads=True, **cfg):
        c = self._cfg(**cfg)
        f = self.lib.mdr_loss_step_cfg
        f.restype = C.c_int
        f.argtypes = [C.POINTER(C.c_int), _f, _f, C.c_int, C.c_int, C.c_int, _f, C.c_float,
                      C.c_int, C.POINTER(C.c_double), _f, _f]
        l, w, h = fixed.shape[1:]
        loss = C.c_double()
        gp = np.zeros_like(packed) if grads else None
        phi = np.zeros((3, l, w, h), np.float32)
        if f(c, _fp(fixed), _fp(moving), h, w, l, _fp(packed), lam, window, C.byref(loss),
             _fp(gp), _fp(phi)):
            raise RuntimeError(self._perr().decode())
        return loss.value, gp, phi

    def pairwise_optimize_cfg(self, fixed, moving, lf, lm, packed, iters, lr=1e-4, lam=1.0,
                              window=9, optimizer="adam", **cfg):
        c = self._cfg(**cfg)
        f = self.lib.mdr_pairwise_optimize_cfg
        f.restype = C.c_int
        f.argtypes = [C.POINTER(C.c_int), C.c_int, _f, _f, _i, _i, C.c_int, C.c_int, C.c_int,
                      _f, C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double),
                      C.POINTER(C.c_double), _f]
        l, w, h = fixed.shape[1:]
        lt = (C.c_double * (iters + 1))()
        dt = (C.c_double * (iters + 1))()
        phi = np.zeros((3, l, w, h), np.float32)
        ip = lambda a: np.ascontiguousarray(a, np.int32).ctypes.data_as(_i)  # noqa: E731
        if f(c, 0 if optimizer == "adam" else 1, _fp(fixed), _fp(moving), ip(lf), ip(lm), h, w,
             l, _fp(packed), iters, lr, lam, window, lt, dt, _fp(phi)):
            raise RuntimeError(self._perr().decode())
        return list(lt), list(dt), phi

    def level_param_count(self, C_, S, hd, nb=3):
        return int(self._lpc(C_, S, hd, nb))

    # -- attention ---------------------------------------------------------
    def window_offset(self, o, nb=3):
        off = (C.c_int * 3)()
        self._window_offset(o, nb, off)
        return tuple(off)

    def na_fwd(self, Q, K, B, dims, S, hd, nb=3):
        """Returns (W, bad) — bad is None or (x,y,z,head) of the first
        non-finite logit (the reference raises numeric_error there)."""
        h, w, l = dims
        n = h * w * l
        W = np.zeros((S, n, nb ** 3), np.float32)
        if self.prefix == "mdo_":
            bad = (C.c_int * 4)()
            rc = self._na_fwd(_fp(Q), _fp(K), _fp(B), h, w, l, S, hd, nb, _fp(W), bad)
            return W, (tuple(bad) if rc == 1 else None)
        rc = self._na_fwd(_fp(Q), _fp(K), _fp(B), h, w, l, S, hd, nb, _fp(W))
        return W, (self._last_error().decode() if rc else None)

    def na_naive_fwd(self, Q, K, B, dims, S, hd, nb=3):
        h, w, l = dims
        W = np.zeros((S, h * w * l, nb ** 3), np.float32)
        rc = self._na_naive_fwd(_fp(Q), _fp(K), _fp(B), h, w, l, S, hd, nb, _fp(W))
        return W, (self._last_error().decode() if rc else None)

    def na_bwd(self, Q, K, W, gW, dims, S, hd, nb=3, gQ=None, gK=None, gB=None):
        h, w, l = dims
        gQ = np.zeros_like(Q) if gQ is None else gQ
        gK = np.zeros_like(K) if gK is None else gK
        gB = np.zeros((S, nb ** 3), np.float32) if gB is None else gB
        self._na_bwd(_fp(Q), _fp(K), _fp(W), h, w, l, S, hd, nb, _fp(gW), _fp(gQ), _fp(gK),
                     _fp(gB))
        return gQ, gK, gB

    def subfields_fwd(self, W, dims, S, nb=3):
        h, w, l = dims
        out = np.zeros((3 * S, l, w, h), np.float32)
        self._sf_fwd(_fp(W), h, w, l, S, nb, _fp(out))
        return out

    def subfields_bwd(self, gout, dims, S, nb=3, gW=None):
        h, w, l = dims
        gW = np.zeros((S, h * w * l, nb ** 3), np.float32) if gW is None else gW
        self._sf_bwd(h, w, l, S, nb, _fp(gout), _fp(gW))
        return gW

    # -- sampling ----------------------------------------------------------
    def resolve_axis(self, x, dim):
        i0, i1, live = C.c_int(), C.c_int(), C.c_int()
        f = C.c_float()
        self._resolve(C.c_float(x), dim, C.byref(i0), C.byref(i1), C.byref(f), C.byref(live))
        return i0.value, i1.value, f.value, live.value

    def warp_fwd(self, vol, field):
        Cc = vol.shape[0]
        l, w, h = vol.shape[1:]
        out = np.zeros_like(vol)
        self._warp_fwd(_fp(vol), Cc, h, w, l, _fp(field), _fp(out))
        return out

    def warp_bwd(self, vol, field, gout, want_gin=True, want_gfield=True, gin=None, gfield=None):
        Cc = vol.shape[0]
        l, w, h = vol.shape[1:]
        if want_gin and gin is None:
            gin = np.zeros_like(vol)
        if want_gfield and gfield is None:
            gfield = np.zeros_like(field)
        self._warp_bwd(_fp(vol), Cc, h, w, l, _fp(field), _fp(gout),
                       _fp(gin) if want_gin else None, _fp(gfield) if want_gfield else None)
        return gin, gfield

    def upsample_target_ok(self, dims, tdims):
        return bool(self._up_ok(*dims, *tdims))

    def upsample2_fwd(self, x, tdims, scale=2.0):
        Cc = x.shape[0]
        l, w, h = x.shape[1:]
        th, tw, tl = tdims
        out = np.zeros((Cc, tl, tw, th), np.float32)
        self._up_fwd(_fp(x), Cc, h, w, l, th, tw, tl, scale, _fp(out))
        return out

    def upsample2_bwd(self, gout, dims, scale=2.0, gin=None):
        Cc = gout.shape[0]
        tl, tw, th = gout.shape[1:]
        h, w, l = dims
        gin = np.zeros((Cc, l, w, h), np.float32) if gin is None else gin
        self._up_bwd(Cc, h, w, l, th, tw, tl, scale, _fp(gout), _fp(gin))
        return gin

    # -- conv / fields -----------------------------------------------------
    def conv3_fwd(self, x, k, bias):
        ic = x.shape[0]
        l, w, h = x.shape[1:]
        oc = k.shape[0]
        out = np.zeros((oc, l, w, h), np.float32)
        self._conv_fwd(_fp(x), ic, h, w, l, _fp(k), _fp(bias), oc, _fp(out))
        return out

    def conv3_bwd(self, x, k, gout, gin=None, gk=None, gbias=None):
        ic = x.shape[0]
        l, w, h = x.shape[1:]
        oc = k.shape[0]
        gin = np.zeros_like(x) if gin is None else gin
        gk = np.zeros_like(k) if gk is None else gk
        gbias = np.zeros((oc,), np.float32) if gbias is None else gbias
        self._conv_bwd(_fp(x), ic, h, w, l, _fp(k), oc, _fp(gout), _fp(gin), _fp(gk), _fp(gbias))
        return gin, gk, gbias

    def compose_fwd(self, prev, res):
        l, w, h = prev.shape[1:]
        out = np.zeros_like(prev)
        self._comp_fwd(_fp(prev), _fp(res), h, w, l, _fp(out))
        return out

    def compose_bwd(self, prev, res, gout, gprev=None, gres=None):
        l, w, h = prev.shape[1:]
        gprev = np.zeros_like(prev) if gprev is None else gprev
        gres = np.zeros_like(res) if gres is None else gres
        self._comp_bwd(_fp(prev), _fp(res), h, w, l, _fp(gout), _fp(gprev), _fp(gres))
        return gprev, gres

    def scaling_squaring(self, vel, steps):
        l, w, h = vel.shape[1:]
        out = np.zeros_like(vel)
        self._ss(_fp(vel), h, w, l, steps, _fp(out))
        return out

    # -- reference-only helpers --------------------------------------------
    def make_smooth_velocity(self, dims, seed, magnitude, sigma):
        h, w, l = dims
        out = np.zeros((3, l, w, h), np.float32)
        self._smooth_vel(h, w, l, seed, magnitude, sigma, _fp(out))
        return out


class Rng:
    """splitmix64 + Box-Muller stream, bit-identical to reference rng.hpp:23-67
    (vectorised in numpy; ``normal`` honours the one-value cache)."""

    _G = np.uint64(0x9E3779B97F4A7C15)

    def __init__(self, seed: int):
        self.state = np.uint64(seed)
        self.spare = None

    def next_u64(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            k = np.arange(1, n + 1, dtype=np.uint64)
            z = self.state + k * self._G
            self.state = self.state + np.uint64(n) * self._G
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))

    def uniform01(self, n: int) -> np.ndarray:
        return (self.next_u64(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        return lo + (hi - lo) * self.uniform01(n)

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + int(int(self.next_u64(1)[0]) % (hi - lo + 1))

    def normal(self, n: int, mean: float = 0.0, sd: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        i = 0
        if self.spare is not None and n > 0:
            out[0] = self.spare
            self.spare = None
            i = 1
        rem = n - i
        pairs = (rem + 1) // 2
        if pairs:
            u = self.uniform01(2 * pairs)
            u1 = np.maximum(u[0::2], 1e-300)
            u2 = u[1::2]
            r = np.sqrt(-2.0 * np.log(u1))
            a = 6.283185307179586476925286766559 * u2
            vals = np.empty(2 * pairs)
            vals[0::2] = r * np.cos(a)
            vals[1::2] = r * np.sin(a)
            out[i:] = vals[:rem]
            if rem % 2 == 1:
                self.spare = vals[-1]
        return mean + sd * out


_cache = {}


def mdo() -> _Lib:
    if "mdo" not in _cache:
        if not os.path.exists(LIB_MDO):
            build()
        _cache["mdo"] = _Lib(LIB_MDO, "mdo_")
    return _cache["mdo"]


def ref_available() -> bool:
    return os.path.exists(LIB_REF)


def ref() -> _Lib:
    if "ref" not in _cache:
        _cache["ref"] = _Lib(LIB_REF, "mdr_")
    return _cache["ref"]


def _host_isa() -> str:
    """x86-64 micro-architecture level of this host: v4 (AVX-512 F/BW/CD/DQ/VL)
    or v3 (AVX2 + FMA + BMI2), else '' (neither fast build can run)."""
    try:
        flags = set()
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    flags = set(line.split(":", 1)[1].split())
                    break
    except OSError:
        return ""
    if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags:
        return "v4"
    if {"avx2", "fma", "bmi2", "movbe"} <= flags:
        return "v3"
    return ""


def ref_fast_path() -> str:
    """The -O3 native-ISA reference build for this host (BASELINE.md §4 flags),
    else the pinned -O2 build."""
    isa = _host_isa()
    for level in (("v4", "v3") if isa == "v4" else (("v3",) if isa == "v3" else ())):
        p = os.path.join(HERE, "_ref", f"libmdreg_ref_fast_{level}.so")
        if os.path.exists(p):
            return p
    return LIB_REF


def ref_fast() -> _Lib:
    """The reference compiled as BASELINE.md §4 times it (-O3, native ISA):
    the bench's CPU baseline and reference arm.  Not bit-pinned (FP
    contraction on), so parity tests use ref()."""
    if "ref_fast" not in _cache:
        _cache["ref_fast"] = _Lib(ref_fast_path(), "mdr_")
    return _cache["ref_fast"]
