"""Diagnose the deterministic gin gather against the atomic scatter on the
pipelined-host test inputs (nonfinite case)."""
import os, sys, ctypes as C_
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np, torch
from paper_2403_16526_b200 import ops, _capi
dims = (128, 96, 100); h, w, l = dims
for C in (3,):
    r = np.random.default_rng(C)
    vol = r.standard_normal((C, l, w, h)).astype(np.float32)
    fld = r.uniform(-2.5, 2.5, (3, l, w, h)).astype(np.float32)
    fld[2, 40, 3, 5] = np.nan
    fld[0, 60, 7, 9] = np.inf
    g = r.standard_normal((C, l, w, h)).astype(np.float32)
    d = lambda a: torch.from_numpy(a).cuda()
    gin_d, _ = ops.warp_bwd(d(vol), d(fld), d(g))
    gin_d = gin_d.cpu().numpy()
    L = _capi.lib(); p = lambda a: a.ctypes.data_as(C_.c_void_p)
    gin = np.zeros_like(vol); gf = np.zeros((3, l, w, h), np.float32)
    assert L.mdg_warp_bwd_host(p(vol), C, _capi.Dims3(*dims), p(fld), p(g), p(gin), p(gf)) == 0
    bad = ~np.isclose(gin, gin_d, rtol=1e-4, atol=1e-5, equal_nan=True)
    print("C", C, "mismatches", bad.sum(), "nan dev", np.isnan(gin_d).sum(), "nan host", np.isnan(gin).sum())
    idx = np.argwhere(bad)[:10]
    for i in idx: print(tuple(i), gin[tuple(i)], gin_d[tuple(i)])
    # whole-volume range calls on device vs atomic env
    os.environ["MDG_WARP_ATOMIC"] = "1"
