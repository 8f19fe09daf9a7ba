"""Per-launch device time (with grid) of the encoder forward+backward of one
image at 160x192x224, from a chrome trace of the torch profiler."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2403_16526_b200 import ops
h, w, l = 160, 192, 224
params = [t.cuda() for t in ops.init_model(42)]
blocks = [ops.BlockParams(*params[8 * k:8 * k + 8]) for k in range(5)]
grads = [torch.zeros_like(t) for t in params[:40]]
gblocks = [ops.BlockParams(*grads[8 * k:8 * k + 8]) for k in range(5)]
enc = ops.Encoder((h, w, l))
img = ops.Rng(11).uniform((1, l, w, h)).cuda()
def run():
    feats = enc.forward(img, blocks)
    enc.backward([torch.ones_like(f) * 1e-3 for f in feats], gblocks)
for _ in range(2): run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run(); torch.cuda.synchronize()
path = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(path)
tr = json.load(open(path))
tot = 0.0
for e in tr["traceEvents"]:
    if e.get("cat") == "kernel":
        nm = e["name"].replace("void ", "").replace("(anonymous namespace)::", "").split("(")[0][-34:]
        a = e.get("args", {})
        tot += e["dur"]
        if e["dur"] > 20:
            print(f"{nm:34s} {str(a.get('grid')):18s} {str(a.get('block')):14s} {e['dur']:8.1f} us")
print(f"total {tot/1e3:.2f} ms")
