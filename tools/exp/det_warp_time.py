"""Deterministic-mode warp backward at the bench workload (C = 8, smooth
field): per-kernel split via torch profiler (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

h, w, l = 160, 192, 224
C = 8
vol = torch.randn(C, l, w, h, device="cuda")
field = ops.make_smooth_velocity((h, w, l), 11, 2.0, 4.0).cuda()
gout = torch.randn(C, l, w, h, device="cuda")
gin, gf = torch.zeros_like(vol), torch.zeros_like(field)
ops.set_deterministic(True)
for _ in range(3):
    ops.warp_bwd(vol, field, gout, gin=gin, gfield=gf)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        ops.warp_bwd(vol, field, gout, gin=gin, gfield=gf)
    torch.cuda.synchronize()
for ev in prof.key_averages():
    if ev.device_type.name == "CUDA" or ev.self_device_time_total > 0:
        print(f"{ev.key[:60]:60s} {ev.count:3d} {ev.self_device_time_total / ev.count:9.1f} us")
