"""project_qk fwd+bwd at one level size (ncu target). usage: prof_project.py C K h w l"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402
from paper_2403_16526_b200._capi import MDG_QK_PLANAR  # noqa: E402

C, K, h, w, l = (int(a) for a in sys.argv[1:6]) if len(sys.argv) > 5 else (8, 6, 160, 192, 224)
f = torch.randn(C, l, w, h, device="cuda")
m = torch.randn_like(f)
p = ops.ProjectionParams(torch.randn(K, C, device="cuda"), torch.zeros(K, device="cuda"),
                         torch.ones(K, device="cuda"), torch.zeros(K, device="cuda"))
g = ops.ProjectionParams(*[torch.zeros_like(t) for t in (p.weight, p.bias, p.ln_gamma, p.ln_beta)])
gf, gm = torch.zeros_like(f), torch.zeros_like(m)
for i in range(4):
    Q, Kt = ops.project_qk(f, m, p, layout=MDG_QK_PLANAR)
    ops.project_qk_bwd(f, m, p, Q, Kt, layout=MDG_QK_PLANAR, gf=gf, gm=gm, grads=g)
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
tf, tb = [], []
for _ in range(7):
    e0.record()
    Q, Kt = ops.project_qk(f, m, p, layout=MDG_QK_PLANAR)
    e1.record()
    ops.project_qk_bwd(f, m, p, Q, Kt, layout=MDG_QK_PLANAR, gf=gf, gm=gm, grads=g)
    e2.record()
    torch.cuda.synchronize()
    tf.append(e0.elapsed_time(e1) * 1e3)
    tb.append(e1.elapsed_time(e2) * 1e3)
tf.sort(); tb.sort()
print(f"C={C} K={K} {h}x{w}x{l}: project fwd {tf[3]:.1f} us (min {tf[0]:.1f})  bwd {tb[3]:.1f} us (min {tb[0]:.1f})")
