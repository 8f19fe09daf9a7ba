"""Loss fwd/bwd timing at 160x192x224 (per-kernel with PROFILE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_16526_b200 import ops
h, w, l = 160, 192, 224
g = torch.Generator(device="cuda").manual_seed(0)
fixed = torch.rand(1, l, w, h, device="cuda", generator=g)
moving = torch.rand(1, l, w, h, device="cuda", generator=g)
phi = torch.randn(3, l, w, h, device="cuda", generator=g) * 0.5
cfg = ops.LossConfig()
for _ in range(3):
    ops.total_loss(fixed, moving, phi, cfg); ops.total_loss_bwd(fixed, moving, phi, cfg)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
gphi = torch.zeros_like(phi); gm = torch.zeros_like(moving)
for _ in range(5):
    e[0].record(); ops.total_loss(fixed, moving, phi, cfg); e[1].record()
    ops.total_loss_bwd(fixed, moving, phi, cfg, gphi=gphi, gmoving=gm); e[2].record()
    torch.cuda.synchronize()
    print(f"loss fwd {e[0].elapsed_time(e[1]):.3f} ms  bwd {e[1].elapsed_time(e[2]):.3f} ms")
if os.environ.get("PROFILE"):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ops.total_loss(fixed, moving, phi, cfg); ops.total_loss_bwd(fixed, moving, phi, cfg)
        torch.cuda.synchronize()
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            print(f"  {ev.name[:60]:60s} {ev.device_time:9.1f} us")
