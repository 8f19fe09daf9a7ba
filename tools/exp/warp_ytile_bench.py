"""32x8-tile warp backward with the cross-warp y merge vs libmdg's warp_bwd
(C = 8, smooth field; dev experiment)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwarp_ytile.so"))
h, w, l = 160, 192, 224
C = 8
vol = torch.randn(C, l, w, h, device="cuda")
gout = torch.randn(C, l, w, h, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731


def t(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for name, field in (("smooth", ops.make_smooth_velocity((h, w, l), 11, 2.0, 4.0).cuda()),):
    rg, rf = torch.zeros_like(vol), torch.zeros_like(field)
    ops.warp_bwd(vol, field, gout, gin=rg, gfield=rf)
    for ym in (0, 1):
        g2, f2 = torch.zeros_like(vol), torch.zeros_like(field)
        lib.ytile_bwd(P(vol), P(field), P(gout), h, w, l, P(g2), P(f2), ym, 1, st)
        torch.cuda.synchronize()
        print(name, "ym", ym, "gin rel", float((g2 - rg).abs().max() / rg.abs().max()),
              "gfield rel", float((f2 - rf).abs().max() / rf.abs().max()))
        print(name, "ym", ym, "gin-only ms", round(t(lambda: lib.ytile_bwd(P(vol), P(field), P(gout), h, w, l, P(g2), P(f2), ym, 0, st)), 4),
              "gin+gfield ms", round(t(lambda: lib.ytile_bwd(P(vol), P(field), P(gout), h, w, l, P(g2), P(f2), ym, 1, st)), 4))
    print(name, "libmdg gin-only ms", round(t(lambda: ops.warp_bwd(vol, field, gout, gin=rg, want_gfield=False)), 4),
          "combined ms", round(t(lambda: ops.warp_bwd(vol, field, gout, gin=rg, gfield=rf)), 4))
