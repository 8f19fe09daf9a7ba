"""64-bit fixed-point gin scatter (order-independent integer REDs) vs the fp32
RED scatter at the bench workload (C = 8, smooth field; dev experiment)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwarp_fix.so"))
h, w, l = 160, 192, 224
n = h * w * l
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


for name, field in (("smooth", ops.make_smooth_velocity((h, w, l), 11, 2.0, 4.0).cuda()),
                    ("random", (torch.rand(3, l, w, h, device="cuda") * 4 - 2))):
    ref = torch.zeros_like(vol)
    ops.warp_bwd(vol, field, gout, gin=ref, want_gfield=False)
    mx = torch.zeros(C, dtype=torch.int32, device="cuda")
    acc = torch.zeros(C, n, dtype=torch.int64, device="cuda")
    gf = torch.zeros_like(vol)
    gi = torch.zeros_like(vol)
    lib.fix_scatter(P(field), P(gout), h, w, l, P(gf), P(acc), P(mx), 0, st)
    lib.fix_maxabs(P(gout), C, n, P(mx), st)
    lib.fix_scatter(P(field), P(gout), h, w, l, P(gi), P(acc), P(mx), 1, st)
    lib.fix_convert(P(acc), C, n, P(mx), P(gi), st)
    gi2 = torch.zeros_like(vol)
    lib.fix_scatter(P(field), P(gout), h, w, l, P(gi2), P(acc), P(mx), 1, st)
    lib.fix_convert(P(acc), C, n, P(mx), P(gi2), st)
    torch.cuda.synchronize()
    den = ref.abs().max()
    print(name, "float rel", float((gf - ref).abs().max() / den), "fix rel",
          float((gi - ref).abs().max() / den), "fix repeat identical", bool(torch.equal(gi, gi2)))
    print(name, "libmdg gin-only ms", round(t(lambda: ops.warp_bwd(vol, field, gout, gin=gf, want_gfield=False)), 4))
    print(name, "float scatter ms", round(t(lambda: lib.fix_scatter(P(field), P(gout), h, w, l, P(gf), P(acc), P(mx), 0, st)), 4))
    print(name, "maxabs ms", round(t(lambda: lib.fix_maxabs(P(gout), C, n, P(mx), st)), 4))
    print(name, "fix scatter ms", round(t(lambda: lib.fix_scatter(P(field), P(gout), h, w, l, P(gi), P(acc), P(mx), 1, st)), 4))
    print(name, "convert ms", round(t(lambda: lib.fix_convert(P(acc), C, n, P(mx), P(gi), st)), 4))
    with_det = ops.set_deterministic(True)
    print(name, "libmdg deterministic gin-only ms", round(t(lambda: ops.warp_bwd(vol, field, gout, gin=gf, want_gfield=False)), 4))
    ops.set_deterministic(with_det)
