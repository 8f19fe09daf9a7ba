import os, sys, time, types
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2403_16526_b200 import _capi, ops
L = _capi.lib()
host_in = bench.make_inputs(0)
h, w, l = bench.DIMS
n = h * w * l
S, HD, CH = bench.S, bench.HD, bench.CH
pin = {k: v.pin_memory() for k, v in host_in.items()}
outs = {"SF": torch.empty(3 * S, n).pin_memory(), "LSE": torch.empty(S, n).pin_memory(),
        "gQ": torch.zeros(n, S * HD).pin_memory(), "gK": torch.zeros(n, S * HD).pin_memory(),
        "gB": torch.zeros(S, 27).pin_memory(), "warped": torch.empty(CH, l, w, h).pin_memory(),
        "gin": torch.zeros(CH, l, w, h).pin_memory(), "gfield": torch.zeros(3, l, w, h).pin_memory()}
d3 = ops.dims3(bench.DIMS)
p = lambda t: t.data_ptr()
calls = [
 lambda: L.mdg_modet_fwd_host(p(pin["Q"]), p(pin["K"]), p(pin["B"]), d3, S, HD, 3, 1, p(outs["SF"]), p(outs["LSE"])),
 lambda: L.mdg_modet_bwd_host(p(pin["Q"]), p(pin["K"]), p(pin["B"]), p(outs["SF"]), p(outs["LSE"]), p(pin["gSF"]), d3, S, HD, 3, 1, p(outs["gQ"]), p(outs["gK"]), p(outs["gB"]), 0),
 lambda: L.mdg_warp_fwd_host(p(pin["feat"]), CH, d3, p(pin["field"]), p(outs["warped"])),
 lambda: L.mdg_warp_bwd_host(p(pin["feat"]), CH, d3, p(pin["field"]), p(pin["gout"]), p(outs["gin"]), p(outs["gfield"])),
]
for rep in range(int(os.environ.get("REPS", "6"))):
    tt = []
    for fn in calls:
        t1 = time.perf_counter(); assert fn() == 0; tt.append(round((time.perf_counter() - t1) * 1e3, 2))
    print(rep, round(sum(tt), 1), tt)
