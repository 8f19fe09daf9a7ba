"""mdg_encoder_conv3_fwd / input gradient at the encoder's L1-L4 shapes:
device time and relative error vs float64 (run with MDG_ENC_TC=0 and =1)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import _capi, ops  # noqa: E402

L = _capi.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
F = torch.nn.functional


def t(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
tag = os.environ.get("MDG_ENC_TC", "1")
for (h, w, l), ic, oc in (((40, 48, 56), 16, 32), ((40, 48, 56), 32, 32), ((20, 24, 28), 32, 64),
                          ((20, 24, 28), 64, 64), ((10, 12, 14), 64, 128),
                          ((10, 12, 14), 128, 128)):
    n = h * w * l
    g = torch.Generator(device="cuda").manual_seed(ic * 7 + oc)
    x = torch.randn(ic, n, device="cuda", generator=g)
    wt = torch.randn(oc, ic, 3, 3, 3, device="cuda", generator=g) / (ic * 27) ** 0.5
    b = torch.randn(oc, device="cuda", generator=g)
    gout = torch.randn(oc, n, device="cuda", generator=g)
    out = torch.empty(oc, n, device="cuda")
    gin = torch.zeros(ic, n, device="cuda")
    d3 = ops.dims3((h, w, l))
    fwd = lambda: L.mdg_encoder_conv3_fwd(P(x), ic, d3, P(wt), P(b), oc, P(out), st)  # noqa: E731
    bwd = lambda: L.mdg_encoder_conv3_bwd(P(x), ic, d3, P(wt), oc, P(gout), P(gin), None, None, st)  # noqa: E731
    assert fwd() == 0
    gin.zero_()
    assert bwd() == 0
    torch.cuda.synchronize()
    xr = x.double().view(1, ic, l, w, h).requires_grad_(True)
    r = F.conv3d(xr, wt.double(), b.double(), padding=1)
    r.backward(gout.double().view(1, oc, l, w, h))
    e_f = float((out.double() - r.view(oc, n)).norm() / r.norm())
    e_b = float((gin.double() - xr.grad.view(ic, n)).norm() / xr.grad.norm())
    tf, tb = t(fwd), t(bwd)
    print(f"TC={tag} {h}x{w}x{l} {ic}->{oc}: fwd {tf:6.1f} us err {e_f:.1e} | gin {tb:6.1f} us err {e_b:.1e}")
