"""project_qk backward at the L1 shape (C = 8, K = 6, 160x192x224, both
inputs, planar) — device time (dev experiment)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

n = 160 * 192 * 224
C, K = 8, 6
f = torch.randn(C, n, device="cuda")
m = torch.randn(C, n, device="cuda")
p = ops.ProjectionParams(torch.randn(K, C, device="cuda") * 0.3, torch.randn(K, device="cuda"),
                         torch.ones(K, device="cuda"), torch.zeros(K, device="cuda"))
gQ = torch.randn(K, n, device="cuda")
gK = torch.randn(K, n, device="cuda")
gf, gm = torch.zeros_like(f), torch.zeros_like(m)
grads = ops.ProjectionParams(*[torch.zeros_like(t) for t in (p.weight, p.bias, p.ln_gamma, p.ln_beta)])


def run():
    ops.project_qk_bwd(f, m, p, gQ, gK, layout=ops.MDG_QK_PLANAR, gf=gf, gm=gm, grads=grads)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    run()
e1.record()
torch.cuda.synchronize()
print(f"project_qk_bwd L1 {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
