import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np, torch, pyoracle
from _util import f32, rel_norm
from paper_2403_16526_b200 import ops
from test_gpu_encoder import split, device_tensors
ref = pyoracle.ref()
dims = (16, 16, 16); h, w, l = dims
packed, sizes = ref.model_params(42)
r = np.random.default_rng(1)
img = f32(r.uniform(0, 1, (1, l, w, h)))
enc = ops.Encoder(dims)
gfeat = [f32(r.standard_normal((c, d[2], d[1], d[0]))) for c, d in zip(enc.channels, enc.dims)]
feats_r, gp_r, gi_r = ref.encode(img, packed, gfeat)
T = device_tensors(packed, sizes)
blocks = [ops.BlockParams(*T[8 * k:8 * k + 8]) for k in range(5)]
feats = enc.forward(torch.from_numpy(img).cuda(), blocks)
grads = [b.zeros_like() for b in blocks]
gimg = torch.zeros(1, l, w, h, device="cuda")
enc.backward([torch.from_numpy(g).cuda() for g in gfeat], grads, gimg)
torch.cuda.synchronize()
ours = [t.cpu().numpy().ravel() for g in grads for t in g.tensors()]
theirs = split(gp_r, sizes)[:40]
for i, (a, b) in enumerate(zip(ours, theirs)):
    print(i, round(rel_norm(a, b), 6), np.abs(b).max())
print("gimg", rel_norm(gimg.cpu().numpy(), gi_r))
