"""y-pair merged gin scatter vs libmdg's warp_bwd gin at the bench workload
(C = 8, smooth field, dev experiment)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwarp_ypair.so"))
h, w, l = 160, 192, 224
C = 8
vol = torch.randn(C, l, w, h, device="cuda")
field = ops.make_smooth_velocity((h, w, l), 11, 2.0, 4.0).cuda()
gout = torch.randn(C, l, w, h, device="cuda")
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


ref = torch.zeros_like(vol)
ops.warp_bwd(vol, field, gout, gin=ref, want_gfield=False)
gin = torch.zeros_like(vol)
P = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
lib.ypair_gin(P(field), P(gout), h, w, l, P(gin), ctypes.c_void_p(st))
torch.cuda.synchronize()
d = (gin - ref).abs()
print("max |diff|", float(d.max()), "rel", float(d.max() / ref.abs().max()))
g2 = torch.zeros_like(vol)
print("libmdg gin-only ms", round(t(lambda: ops.warp_bwd(vol, field, gout, gin=g2, want_gfield=False)), 4))
print("y-pair gin ms", round(t(lambda: lib.ypair_gin(P(field), P(gout), h, w, l, P(gin),
                                                     ctypes.c_void_p(st))), 4))

lq = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwarp_quad.so"))
gq = torch.zeros_like(vol)
lq.quad_gin(P(field), P(gout), h, w, l, P(gq), ctypes.c_void_p(st))
torch.cuda.synchronize()
d = (gq - ref).abs()
print("quad max |diff|", float(d.max()), "rel", float(d.max() / ref.abs().max()))
print("quad gin ms", round(t(lambda: lq.quad_gin(P(field), P(gout), h, w, l, P(gq),
                                                 ctypes.c_void_p(st))), 4))

for mb in (2, 3, 4):
    print(f"y-pair minb={mb} ms", round(t(lambda: lib.ypair_gin_b(P(field), P(gout), h, w, l, P(gin), mb,
                                                                ctypes.c_void_p(st))), 4))

# gfield-only (libmdg) and the y-pair gin (experiment) on two streams at once
s2 = torch.cuda.Stream()
gf = torch.zeros_like(field)


def both_streams():
    cur = torch.cuda.current_stream()
    s2.wait_stream(cur)
    ops.warp_bwd(vol, field, gout, gfield=gf, want_gin=False)
    lib.ypair_gin_b(P(field), P(gout), h, w, l, P(gin), 4, ctypes.c_void_p(s2.cuda_stream))
    cur.wait_stream(s2)


print("gfield (stream 1) + y-pair gin (stream 2) ms", round(t(both_streams), 4))
print("libmdg combined ms", round(t(lambda: ops.warp_bwd(vol, field, gout, gin=g2, gfield=gf)), 4))
