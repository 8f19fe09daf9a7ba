"""Time individual libmdg ops at the bench size with CUDA events (dev tool).
usage: python tools/bench_ops.py [substring-filter ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_16526_b200 import ops, _capi
try:
    import pynvml; pynvml.nvmlInit(); NV = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    NV = None
L = _capi.lib()
h, w, l = 160, 192, 224
n = h * w * l
C = 8
dev = torch.device("cuda")
feat = torch.randn(C, l, w, h, device=dev)
zz, yy, xx = torch.meshgrid(torch.arange(l, device=dev, dtype=torch.float32), torch.arange(w, device=dev, dtype=torch.float32), torch.arange(h, device=dev, dtype=torch.float32), indexing="ij")
field = torch.stack([2 * torch.sin(xx / 23) * torch.cos(yy / 29), 2 * torch.cos(xx / 27) * torch.sin(zz / 19), 2 * torch.sin(yy / 21) * torch.cos(zz / 17)]).contiguous()
gout = torch.randn_like(feat)
gin = torch.zeros_like(feat); gf = torch.zeros_like(field); out = torch.empty_like(feat)
d3 = ops.dims3((h, w, l)); st = torch.cuda.current_stream().cuda_stream
P = lambda t: t.data_ptr() if t is not None else None
S, D = 1, 6
Q = torch.rand(S * D, n, device=dev) * 2 - 1; K = torch.rand_like(Q) * 2 - 1; B = torch.rand(S, 27, device=dev) - 0.5
SF = torch.empty(3 * S, n, device=dev); LSE = torch.empty(S, n, device=dev); g = torch.rand_like(SF)
gQ = torch.empty_like(Q); gK = torch.empty_like(K); gB = torch.zeros_like(B)
f3 = field.clone(); o3 = torch.empty_like(field)
filt = sys.argv[1:]

def timeit(name, fn, reps=30):
    if filt and not any(f in name for f in filt): return
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record()
    clk = pynvml.nvmlDeviceGetClockInfo(NV, pynvml.NVML_CLOCK_SM) if NV else -1
    torch.cuda.synchronize()
    print(f"{name:32s} {a.elapsed_time(b) / reps * 1e3:8.1f} us   (sm {clk} MHz)", flush=True)

for rnd in range(2):
    timeit("modet_fwd", lambda: L.mdg_modet_fwd(P(Q), P(K), P(B), d3, S, D, 3, 1, P(SF), P(LSE), None, st))
    timeit("modet_bwd row", lambda: L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(g), d3, S, D, 3, 1, P(gQ), None, P(gB), 0, st))
    timeit("modet_bwd col", lambda: L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(g), d3, S, D, 3, 1, None, P(gK), None, 0, st))
    timeit("modet_bwd row+col", lambda: L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(g), d3, S, D, 3, 1, P(gQ), P(gK), P(gB), 0, st))
    timeit("warp_fwd C=8", lambda: L.mdg_warp_fwd(P(feat), C, d3, P(field), P(out), st))
    timeit("warp_bwd C=8", lambda: L.mdg_warp_bwd(P(feat), C, d3, P(field), P(gout), P(gin), P(gf), st))
    timeit("warp_bwd C=8 gin", lambda: L.mdg_warp_bwd(P(feat), C, d3, P(field), P(gout), P(gin), None, st))
    timeit("warp_bwd C=8 gfield", lambda: L.mdg_warp_bwd(P(feat), C, d3, P(field), P(gout), None, P(gf), st))
    timeit("compose_fwd", lambda: L.mdg_compose_fwd(P(field), P(f3), d3, P(o3), st))
    timeit("compose_bwd", lambda: L.mdg_compose_bwd(P(field), P(f3), d3, P(o3), P(gf), P(o3), st))
    timeit("copy 8ch (torch)", lambda: out.copy_(feat))
