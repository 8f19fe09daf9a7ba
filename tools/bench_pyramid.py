"""Time the decoding pyramid (forward, backward) at a given fine size with the
small preset (heads 8,4,2,1,1, hd 6, channels 128..8) on synthetic features.
usage: python tools/bench_pyramid.py [h w l] [--diffeo]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_16526_b200 import ops

args = [a for a in sys.argv[1:] if not a.startswith("--")]
fine = tuple(int(a) for a in args[:3]) if args else (160, 192, 224)
diffeo = "--diffeo" in sys.argv
L = 5
dims = [fine]
for _ in range(L - 1):
    dims.append(tuple((v + 1) // 2 for v in dims[-1]))
dims = dims[::-1]
chans = (128, 64, 32, 16, 8)
heads = (8, 4, 2, 1, 1)
hd = 6
g = torch.Generator(device="cuda").manual_seed(0)
ff = [torch.randn(c, d[2], d[1], d[0], device="cuda", generator=g) for c, d in zip(chans, dims)]
mf = [torch.randn(c, d[2], d[1], d[0], device="cuda", generator=g) for c, d in zip(chans, dims)]
lps = []
for c, S in zip(chans, heads):
    K = S * hd
    lps.append(ops.LevelParams(
        ops.ProjectionParams(torch.randn(K, c, device="cuda") * 0.3, torch.zeros(K, device="cuda"),
                             torch.ones(K, device="cuda"), torch.zeros(K, device="cuda")),
        torch.randn(S, 27, device="cuda") * 0.5, torch.randn(3, 3 * S, 3, 3, 3, device="cuda") * 0.01,
        torch.zeros(3, device="cuda")))
cfg = ops.ModelConfig(heads_per_level=heads, head_dim=hd, diffeomorphic=diffeo)
for check in (True, False):
    pyr = ops.Pyramid(cfg, dims, chans, check_finite=check)
    gphi = torch.randn(3, fine[2], fine[1], fine[0], device="cuda", generator=g)
    grads = [p.zeros_like() for p in lps]
    gf = [torch.zeros_like(t) for t in ff]
    gm = [torch.zeros_like(t) for t in mf]
    for _ in range(3):
        pyr.forward(ff, mf, lps)
        pyr.backward(gphi, grads, gf, gm)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    reps = int(os.environ.get("REPS", "10"))
    tf = tb = 0.0
    for _ in range(reps):
        e[0].record()
        pyr.forward(ff, mf, lps)
        e[1].record()
        pyr.backward(gphi, grads, gf, gm)
        e[2].record()
        torch.cuda.synchronize()
        tf += e[0].elapsed_time(e[1])
        tb += e[1].elapsed_time(e[2])
    print(f"pyramid {fine} diffeo={diffeo} check_finite={check}: fwd {tf/reps:.3f} ms  bwd {tb/reps:.3f} ms  "
          f"arena {pyr.device_bytes/2**20:.0f} MiB")

if os.environ.get("PROFILE"):
    from torch.profiler import profile, ProfilerActivity
    pyr = ops.Pyramid(cfg, dims, chans, check_finite=False)
    pyr.forward(ff, mf, lps); pyr.backward(gphi, grads, gf, gm)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        pyr.forward(ff, mf, lps)
        pyr.backward(gphi, grads, gf, gm)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))
    if os.environ.get("PROFILE") == "2":
        for ev in prof.events():
            if ev.device_type.name == "CUDA":
                print(f"  {ev.name[:60]:60s} {ev.device_time:9.1f} us")
