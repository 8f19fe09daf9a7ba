"""CPU-side op breakdown of one slab PO iteration (torch profiler, aten ops
with CUDA time) — where the torch glue spends its kernels (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2403_16526_b200 import ops, slab_po  # noqa: E402

DIMS = (160, 192, 224)
params = [t.cuda() for t in ops.init_model(42)]
f, m, _, _, _ = ops.synth_pair(DIMS, seed=1, max_disp=2.0)
model = slab_po.SlabModel(params, DIMS)
fl, ml = model.local(f.cuda()), model.local(m.cuda())
for _ in range(2):
    model.po_step(fl, ml)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    model.po_step(fl, ml)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=50))
