"""Warp backward (C = 8) and compose backward at 160x192x224, default vs
deterministic mode, CUDA events; plus one PO iteration (CUDA graph) in each
mode (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402


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


dims = h, w, l = 160, 192, 224
C = 8
vol = torch.randn(C, l, w, h, device="cuda")
gout = torch.randn(C, l, w, h, device="cuda")
gin = torch.zeros_like(vol)
res = ops.make_smooth_velocity(dims, 11, 2.0, 4.0).cuda()
prev = ops.make_smooth_velocity(dims, 12, 2.0, 4.0).cuda()
gf = torch.zeros_like(res)
for name, field in (("smooth", res), ("random", torch.rand(3, l, w, h, device="cuda") * 4 - 2)):
    for det in (False, True):
        ops.set_deterministic(det)
        ms = t(lambda: ops.warp_bwd(vol, field, gout, gin=gin, gfield=gf))
        print(f"warp_bwd C=8 {name} deterministic={det}: {ms:.4f} ms")
for det in (False, True):
    ops.set_deterministic(det)
    ms = t(lambda: ops.compose_bwd(prev, res, res))
    print(f"compose_bwd deterministic={det}: {ms:.4f} ms")
model = ops.NativeModel([p.cuda() for p in ops.init_model(42)], dims)
f, m, _, _, _ = ops.synth_pair(dims, seed=1, max_disp=2.0)
f, m = f.cuda(), m.cuda()
for det in (False, True):
    ops.set_deterministic(det)
    model.po_step(f, m, graph=True)
    ms = t(lambda: model.po_step(f, m, graph=True), k=10)
    print(f"PO iteration deterministic={det}: {ms:.3f} ms")
ops.set_deterministic(False)
