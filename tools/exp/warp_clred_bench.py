"""Channel-last vector-RED gin scatter vs libmdg's warp_bwd gin at the bench
workload (C = 8, smooth field); also checks the result (dev experiment)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwarp_clred.so"))
h, w, l = 160, 192, 224
C = 8
n = h * w * l
vol = torch.randn(C, l, w, h, device="cuda")
field = ops.make_smooth_velocity((h, w, l), 11, 2.0, 4.0).cuda()
gout = torch.randn(C, l, w, h, device="cuda")
gcl = torch.zeros(n * 8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


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


gin_ref = torch.zeros_like(vol)
ops.warp_bwd(vol, field, gout, gin=gin_ref, want_gfield=False)
gin = torch.zeros_like(vol)
lib.scatter_cl(ctypes.c_void_p(field.data_ptr()), ctypes.c_void_p(gout.data_ptr()), h, w, l,
               ctypes.c_void_p(gcl.data_ptr()), ctypes.c_void_p(gin.data_ptr()), 6,
               ctypes.c_void_p(st))
torch.cuda.synchronize()
print("max |diff|", float((gin - gin_ref).abs().max()), "ref max", float(gin_ref.abs().max()))
g2 = torch.zeros_like(vol)
print("libmdg gin-only ms", round(t(lambda: ops.warp_bwd(vol, field, gout, gin=g2, want_gfield=False)), 4))
for mb in (4, 6, 8):
    print(f"cl-red total (memset+scatter+add) minb={mb} ms",
          round(t(lambda: lib.scatter_cl(ctypes.c_void_p(field.data_ptr()),
                                          ctypes.c_void_p(gout.data_ptr()), h, w, l,
                                          ctypes.c_void_p(gcl.data_ptr()),
                                          ctypes.c_void_p(gin.data_ptr()), mb,
                                          ctypes.c_void_p(st))), 4))
print("cl-red scatter only ms",
      round(t(lambda: lib.scatter_only(ctypes.c_void_p(field.data_ptr()),
                                        ctypes.c_void_p(gout.data_ptr()), h, w, l,
                                        ctypes.c_void_p(gcl.data_ptr()), ctypes.c_void_p(st))), 4))
