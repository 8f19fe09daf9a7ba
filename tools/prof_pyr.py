"""Per-kernel device time of the decoder pyramid's backward at 160x192x224
(torch profiler), kernel names aggregated."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import bench
from paper_2403_16526_b200 import ops
dev = torch.device("cuda")
# reuse the bench's pyramid setup
pyr_fn = bench.run_pyramid
import inspect
src = inspect.getsource(pyr_fn)
h, w, l = bench.DIMS
cfg = ops.ModelConfig()
params = [t.to(dev) for t in ops.init_model(42)]
model = ops.NativeModel(params, bench.DIMS)
r = ops.Rng(11)
f = r.uniform((1, l, w, h)).cuda(); m = r.uniform((1, l, w, h)).cuda()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3): model.po_step(f, m, graph=False)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        model.po_step(f, m, graph=False); torch.cuda.synchronize()
agg = collections.defaultdict(float); cnt = collections.Counter()
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        k = ev.name.replace("void ", "").replace("(anonymous namespace)::", "").split("(")[0][-46:]
        agg[k] += ev.device_time; cnt[k] += 1
enc = sum(v for k, v in agg.items() if "enc::" in k)
tot = sum(agg.values())
print(f"total kernel time {tot/1e3:.2f} ms (encoder {enc/1e3:.2f} ms, rest {(tot-enc)/1e3:.2f} ms)")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    if "enc::" in k: continue
    print(f"{k:46s} {cnt[k]:4d} {v/1e3:7.3f} ms")
