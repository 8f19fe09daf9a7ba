"""Kernel time breakdown of one depth-slab PO iteration at N = 1 (dev tool)."""
import collections
import os
import sys
import time

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
t = time.perf_counter()
model.po_step(fl, ml)
torch.cuda.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t):.2f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    model.po_step(fl, ml)
    torch.cuda.synchronize()
agg, cnt = collections.defaultdict(float), collections.Counter()
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        k = ev.name.split("(")[0][:60]
        agg[k] += ev.device_time
        cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:30]:
    print(f"{k:60s} {cnt[k]:4d} {v / 1e3:8.2f} ms {100 * v / tot:5.1f}%")
print(f"total kernel time {tot / 1e3:.2f} ms")
