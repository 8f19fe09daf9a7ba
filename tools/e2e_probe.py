"""Per-call timing of the host-buffer drop-ins at the bench size, plus raw
pinned H2D / D2H / duplex copy bandwidth (for the e2e pipelining decision)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2403_16526_b200 import _capi, ops

L = _capi.lib()
h, w, l = bench.DIMS
n = h * w * l
S, HD, CH = bench.S, bench.HD, bench.CH
host = {k: v.pin_memory() for k, v in bench.make_inputs(0).items()}
outs = {"SF": torch.empty(3 * S, n).pin_memory(), "LSE": torch.empty(S, n).pin_memory(),
        "gQ": torch.zeros(S * HD, n).pin_memory(), "gK": torch.zeros(S * HD, n).pin_memory(),
        "gB": torch.zeros(S, 27).pin_memory(), "warped": torch.empty(CH, l, w, h).pin_memory(),
        "gin": torch.zeros(CH, l, w, h).pin_memory(), "gfield": torch.zeros(3, l, w, h).pin_memory()}
d3 = ops.dims3(bench.DIMS)
p = lambda t: t.data_ptr()
calls = {
    "modet_fwd_host": lambda: L.mdg_modet_fwd_host(p(host["Q"]), p(host["K"]), p(host["B"]), d3, S, HD, 3, 1, p(outs["SF"]), p(outs["LSE"])),
    "modet_bwd_host": lambda: L.mdg_modet_bwd_host(p(host["Q"]), p(host["K"]), p(host["B"]), p(outs["SF"]), p(outs["LSE"]), p(host["gSF"]), d3, S, HD, 3, 1, p(outs["gQ"]), p(outs["gK"]), p(outs["gB"]), 0),
    "warp_fwd_host": lambda: L.mdg_warp_fwd_host(p(host["feat"]), CH, d3, p(host["field"]), p(outs["warped"])),
    "warp_bwd_host": lambda: L.mdg_warp_bwd_host(p(host["feat"]), CH, d3, p(host["field"]), p(host["gout"]), p(outs["gin"]), p(outs["gfield"])),
}
for name, fn in calls.items():
    fn()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); assert fn() == 0; ts.append(time.perf_counter() - t0)
    print(f"{name:16s} {min(ts)*1e3:8.2f} ms")
big = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
big2 = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
dbuf2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(fn, nbytes, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return nbytes * reps / (time.perf_counter() - t0) / 1e9
print("H2D GB/s", round(bw(lambda: dbuf.copy_(big, non_blocking=True), 256 << 20), 1))
print("D2H GB/s", round(bw(lambda: big.copy_(dbuf, non_blocking=True), 256 << 20), 1))
def duplex():
    with torch.cuda.stream(s1): dbuf.copy_(big, non_blocking=True)
    with torch.cuda.stream(s2): big2.copy_(dbuf2, non_blocking=True)
print("duplex GB/s (sum of both directions)", round(bw(duplex, 2 * (256 << 20)), 1))
seq = list(calls.values())
for rep in range(4):
    t0 = time.perf_counter()
    tt = []
    for fn in seq:
        t1 = time.perf_counter(); assert fn() == 0; tt.append((time.perf_counter() - t1) * 1e3)
    print("sequence", round((time.perf_counter() - t0) * 1e3, 2), "ms", [round(x, 2) for x in tt])
