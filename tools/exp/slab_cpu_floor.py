"""Host-side floor of one eager slab PO iteration: the same step on a tiny
volume (GPU work negligible), fixed reach and data-dependent (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops, slab_po  # noqa: E402

dims = (32, 32, 32)
params = [t.cuda() for t in ops.init_model(42)]
f, m, _, _, _ = ops.synth_pair(dims, seed=1, max_disp=2.0)
f, m = f.cuda(), m.cuda()
for reach in (None, 6):
    model = slab_po.SlabModel(params, dims, reach=reach)
    for _ in range(3):
        model.po_step(f, m)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        model.po_step(f, m)
    torch.cuda.synchronize()
    print(f"reach={reach}: {1e3 * (time.perf_counter() - t) / 10:.2f} ms per iteration at 32^3")
g = slab_po.SlabModel(params, dims, reach=6)
for _ in range(3):
    g.po_step(f, m, graph=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    g.po_step(f, m, graph=True)
torch.cuda.synchronize()
print(f"graph: {1e3 * (time.perf_counter() - t) / 10:.2f} ms per iteration at 32^3")
