"""Warp backward as one kernel (gin + gfield) versus two launches of the same
kernel (gfield only, gin only) at the bench workload (dev experiment)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

h, w, l = 160, 192, 224
C = 8
vol = torch.randn(C, l, w, h, device="cuda")
field = ops.make_smooth_velocity((h, w, l), 11, 2.0, 4.0).cuda()  # the bench's field
gout = torch.randn(C, l, w, h, device="cuda")
gin = torch.zeros_like(vol)
gf = torch.zeros_like(field)


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


print("field max", float(field.abs().max()))
print("both   ms", t(lambda: ops.warp_bwd(vol, field, gout, gin=gin, gfield=gf)))
print("gfield ms", t(lambda: ops.warp_bwd(vol, field, gout, gfield=gf, want_gin=False)))
print("gin    ms", t(lambda: ops.warp_bwd(vol, field, gout, gin=gin, want_gfield=False)))

for Cc in (1, 2, 4, 8, 16):
    v = torch.randn(Cc, l, w, h, device="cuda")
    go = torch.randn(Cc, l, w, h, device="cuda")
    gi = torch.zeros_like(v)
    print(f"C={Cc:2d} gin-only ms", round(t(lambda: ops.warp_bwd(v, field, go, gin=gi, want_gfield=False)), 4),
          "gfield-only ms", round(t(lambda: ops.warp_bwd(v, field, go, gfield=gf, want_gin=False)), 4))
