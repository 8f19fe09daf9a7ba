import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_16526_b200 import ops, _capi
L = _capi.lib()
h, w, l = 160, 192, 224; n = h * w * l; S, D = 1, 6
dev = torch.device("cuda")
d3 = ops.dims3((h, w, l)); st = torch.cuda.current_stream().cuda_stream
P = lambda t: t.data_ptr() if t is not None else None
Q = torch.rand(S * D, n, device=dev) * 2 - 1; K = torch.rand_like(Q) * 2 - 1; B = torch.rand(S, 27, device=dev) - 0.5
SF = torch.empty(3 * S, n, device=dev); LSE = torch.empty(S, n, device=dev); g = torch.rand_like(SF)
gQ = torch.empty_like(Q); gK = torch.empty_like(K); gB = torch.zeros_like(B)
L.mdg_modet_fwd(P(Q), P(K), P(B), d3, S, D, 3, 1, P(SF), P(LSE), None, st)
row = lambda: L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(g), d3, S, D, 3, 1, P(gQ), None, P(gB), 0, st)
col = lambda: L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(g), d3, S, D, 3, 1, None, P(gK), None, 0, st)
both = lambda: L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(g), d3, S, D, 3, 1, P(gQ), P(gK), P(gB), 0, st)
def timeit(name, fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    print(f"{name:30s} {a.elapsed_time(b) / reps * 1e3:8.1f} us", flush=True)
timeit("row", row); timeit("col", col); timeit("both", both)
timeit("row;col", lambda: (row(), col())); timeit("col;row", lambda: (col(), row()))
timeit("row", row); timeit("col", col); timeit("both", both)
