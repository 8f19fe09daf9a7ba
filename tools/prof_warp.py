"""warp_bwd variants at the bench size (ncu target): MODE=gin|gfield|both"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_16526_b200 import ops, _capi
L = _capi.lib()
h, w, l = 160, 192, 224
C = 8
feat = torch.randn(C, l, w, h, device="cuda")
zz, yy, xx = torch.meshgrid(*(torch.arange(v, device="cuda", dtype=torch.float32) for v in (l, w, h)), indexing="ij")
field = torch.stack([2 * torch.sin(xx / 23) * torch.cos(yy / 29), 2 * torch.cos(xx / 27) * torch.sin(zz / 19),
                     2 * torch.sin(yy / 21) * torch.cos(zz / 17)]).contiguous()
gout = torch.randn_like(feat)
gin = torch.zeros_like(feat); gf = torch.zeros_like(field)
mode = os.environ.get("MODE", "both")
P = lambda t: t.data_ptr() if t is not None else None
d3 = ops.dims3((h, w, l)); st = torch.cuda.current_stream().cuda_stream
a = gin if mode in ("gin", "both") else None
b = gf if mode in ("gfield", "both") else None
for _ in range(5):
    assert L.mdg_warp_bwd(P(feat), C, d3, P(field), P(gout), P(a), P(b), st) == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    L.mdg_warp_bwd(P(feat), C, d3, P(field), P(gout), P(a), P(b), st)
e1.record(); torch.cuda.synchronize()
print(mode, e0.elapsed_time(e1) / 10 * 1e3, "us")
