"""Per-shape device time of the encoder conv (fwd, bwd_in, wgrad) at the
small-preset levels of 160x192x224.  MDG_ENC_ALGO=tiled|igemm forces a path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_16526_b200 import _capi, ops
L = _capi.lib()
dims = [(160, 192, 224)]
for _ in range(4):
    dims.append(ops.halved(dims[-1]))
s = torch.cuda.current_stream().cuda_stream
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
tot = 0.0
for k, d in enumerate(dims):
    n = d[0] * d[1] * d[2]
    c = 8 << k
    for (ic, oc) in [((1 if k == 0 else c // 2), c), (c, c)]:
        if os.environ.get("ONLY") and os.environ["ONLY"] != f"L{k}:{ic}:{oc}":
            continue
        d3 = ops.dims3(d)
        x = torch.randn(ic, n, device="cuda"); w = torch.randn(oc, ic, 27, device="cuda") * 0.1
        b = torch.zeros(oc, device="cuda"); o = torch.empty(oc, n, device="cuda")
        go = torch.randn(oc, n, device="cuda"); gi = torch.zeros(ic, n, device="cuda")
        gw = torch.zeros_like(w); gb = torch.zeros_like(b)
        fw = t(lambda: L.mdg_encoder_conv3_fwd(x.data_ptr(), ic, d3, w.data_ptr(), b.data_ptr(), oc, o.data_ptr(), s))
        bi = t(lambda: L.mdg_encoder_conv3_bwd(x.data_ptr(), ic, d3, w.data_ptr(), oc, go.data_ptr(), gi.data_ptr(), None, None, s))
        bw = t(lambda: L.mdg_encoder_conv3_bwd(x.data_ptr(), ic, d3, w.data_ptr(), oc, go.data_ptr(), None, gw.data_ptr(), gb.data_ptr(), s))
        gf = 2 * n * ic * oc * 27 / 1e9
        tot += fw + bi + bw
        print(f"L{k} {ic:3d}->{oc:3d} n={n:8d}  fwd {fw:7.1f} us ({gf/fw*1e3:5.1f} TF/s)  "
              f"bwd_in {bi:7.1f} us ({gf/bi*1e3:5.1f})  wgrad {bw:7.1f} us ({gf/bw*1e3:5.1f})")
print(f"total {tot/1e3:.2f} ms")
