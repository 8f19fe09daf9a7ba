"""Experiment: channel-last warp forward (tools/exp/warp_cl.cu) vs mdg_warp_fwd."""
import ctypes as C, os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2403_16526_b200 import ops
lib = C.CDLL(os.path.join(ROOT, "tools", "exp", "libwarp_cl.so"))
dims = (160, 192, 224); h, w, l = dims; n = h * w * l
feat = ops.Rng(7).normal((8, l, w, h)).cuda()
fld = ops.make_smooth_velocity(dims, 11, 2.0, 4.0).cuda()
cl = torch.empty(n * 8, device="cuda"); out = torch.empty_like(feat)
st = torch.cuda.current_stream().cuda_stream
ref = ops.warp(feat, fld)
lib.exp_warp_cl(C.c_void_p(feat.data_ptr()), C.c_void_p(cl.data_ptr()), h, w, l, C.c_void_p(fld.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(st), 1)
torch.cuda.synchronize()
print("bit-exact:", torch.equal(out, ref))
def t(fn, reps=20):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3): fn()
    xs = []
    for _ in range(reps):
        e[0].record(); fn(); e[1].record(); torch.cuda.synchronize(); xs.append(e[0].elapsed_time(e[1]))
    return statistics.median(xs)
print("mdg_warp_fwd ms", t(lambda: ops.warp(feat, fld)))
print("cl gather only ms", t(lambda: lib.exp_warp_cl(C.c_void_p(feat.data_ptr()), C.c_void_p(cl.data_ptr()), h, w, l, C.c_void_p(fld.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(st), 0)))
print("cl convert+gather ms", t(lambda: lib.exp_warp_cl(C.c_void_p(feat.data_ptr()), C.c_void_p(cl.data_ptr()), h, w, l, C.c_void_p(fld.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(st), 1)))
