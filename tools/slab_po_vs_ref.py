"""Per-tensor gradient error against the reference's run_loss_step: the
one-slab SlabModel (torch-glue arithmetic) and the native model side by side
(dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import pyoracle  # noqa: E402
from paper_2403_16526_b200 import ops, slab_po  # noqa: E402
from test_gpu_encoder import perturbed_model, shapes, split  # noqa: E402

ref = pyoracle.ref()
dims = tuple(int(v) for v in (sys.argv[1:4] or (32, 32, 32)))
fixed, moving, _, _, _ = ref.synth_pair(dims, seed=3)
packed, sizes = perturbed_model(ref, 5)
params = [np.ascontiguousarray(a.reshape(s)) for a, s in zip(split(packed, sizes), shapes(sizes))]
loss_r, gp_r, phi_r = ref.loss_step(fixed, moving, packed, lam=1.0, window=9)
theirs = split(gp_r, sizes)
sm = slab_po.SlabModel([torch.from_numpy(p).cuda() for p in params], dims)
ts, phs = sm.loss_step(torch.from_numpy(fixed).cuda(), torch.from_numpy(moving).cuda())
nat = ops.NativeModel([torch.from_numpy(p).cuda() for p in params], dims)
tn, phn = nat.loss_step(torch.from_numpy(fixed).cuda(), torch.from_numpy(moving).cuda())
gn = nat.grads


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


print("loss ref", loss_r, "slab", float(ts[0]), "native", float(tn[0]))
print("phi rel slab", rel(phs.cpu(), phi_r), "native", rel(phn.cpu(), phi_r))
for i in range(75):
    print(f"{i:3d} slab {rel(sm.grads[i].cpu(), theirs[i]):.2e} native {rel(gn[i].cpu(), theirs[i]):.2e}"
          f" slab-vs-native {rel(sm.grads[i].cpu(), gn[i].cpu()):.2e}")
