"""tcgen05 3xTF32 implicit-GEMM conv vs libmdg's encoder conv (FFMA2 / igemm):
max relative difference and device time at the encoder's level shapes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import _capi, ops  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcconv.so"))
L = _capi.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


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
for (h, w, l), ic, oc in (((80, 96, 112), 16, 16),
                          ((40, 48, 56), 32, 32), ((40, 48, 56), 16, 32), ((20, 24, 28), 64, 64),
                          ((10, 12, 14), 128, 128)):
    n = h * w * l
    x = torch.randn(ic, n, device="cuda")
    wt = torch.randn(oc, ic, 3, 3, 3, device="cuda") * (1.0 / (ic * 27) ** 0.5)
    b = torch.randn(oc, device="cuda")
    ref = torch.empty(oc, n, device="cuda")
    out = torch.empty(oc, n, device="cuda")
    Kp = (27 * ic + 31) // 32 * 32
    scratch = torch.empty(2 * oc * Kp, device="cuda")
    d3 = ops.dims3((h, w, l))
    go_ref = lambda: L.mdg_encoder_conv3_fwd(P(x), ic, d3, P(wt), P(b), oc, P(ref), st)  # noqa: E731
    go_tc = lambda: lib.tcconv_fwd(P(x), ic, h, w, l, P(wt), P(b), oc, P(out), P(scratch), st)  # noqa: E731
    assert go_ref() == 0 and go_tc() == 0
    torch.cuda.synchronize()
    # float64 reference on a slab of planes
    rel = float((out - ref).abs().max() / ref.abs().max())
    # both against float64 (relative L2 norm, the op test's criterion)
    F = torch.nn.functional
    r64 = F.conv3d(x.double().view(1, ic, l, w, h), wt.double(), b.double(), padding=1).view(oc, n)
    rn = lambda a: float((a.double() - r64).norm() / r64.norm())  # noqa: E731
    tr, tt = t(go_ref), t(go_tc)
    flop = 2.0 * n * 27 * ic * oc
    print(f"{h}x{w}x{l} {ic}->{oc}: relnorm vs f64 libmdg {rn(ref):.2e} tcgen05 {rn(out):.2e}; "
          f"max rel diff {rel:.2e}; libmdg {tr:.1f} us "
          f"({flop / tr / 1e6:.1f} TF/s), tcgen05 3xTF32 {tt:.1f} us ({flop / tt / 1e6:.1f} TF/s)")
