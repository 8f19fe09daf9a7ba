"""One eager PO iteration of the small-preset model at 160x192x224 (native
driver: encoder x2 -> pyramid -> NCC + grad_reg -> backward -> Adam), inside
a cudaProfilerStart/Stop window, after warm-up outside it.  For ncu:

    ncu --profile-from-start off --metrics gpu__time_duration.sum,... \
        python tools/po_iter_once.py

so every kernel of exactly one iteration is captured once (eager launches:
the graph replay runs the same kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402

dims = (160, 192, 224)
model = ops.NativeModel([t.cuda() for t in ops.init_model(42)], dims)
f, m, _, _, _ = ops.synth_pair(dims, seed=1, max_disp=2.0)
f, m = f.cuda(), m.cuda()
for _ in range(2):
    model.po_step(f, m, graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.start()
model.po_step(f, m, graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("po iteration captured")
