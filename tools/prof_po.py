"""Per-kernel device time of one full PO iteration at 160x192x224 (torch profiler)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2403_16526_b200 import ops
h, w, l = 160, 192, 224
model = ops.NativeModel([t.cuda() for t in ops.init_model(42)], (h, w, l))
r = ops.Rng(11)
f = r.uniform((1, l, w, h)).cuda(); m = r.uniform((1, l, w, h)).cuda()
for _ in range(2): model.po_step(f, m)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    model.po_step(f, m); torch.cuda.synchronize()
agg = collections.defaultdict(float); cnt = collections.Counter()
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        k = ev.name.split("(")[0][:50]; agg[k] += ev.device_time; cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:60]:
    print(f"{k:50s} {cnt[k]:4d} {v/1e3:8.2f} ms {100*v/tot:5.1f}%")
print(f"total {tot/1e3:.2f} ms")
if os.environ.get("EVENTS"):
    for ev in prof.events():
        if ev.device_type.name == "CUDA" and os.environ["EVENTS"] in ev.name:
            print(f"  {ev.name[:50]:50s} {ev.device_time:9.1f} us")
