# bisect the tiled ModeT kernels: TMA (h%4==0) vs cp.async (h%4!=0), fwd/row/col
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
case = sys.argv[1] if len(sys.argv) > 1 else None
if case is None:
    for c in ["fwd_cp", "fwd_tma", "row_cp", "row_tma", "col_cp", "col_tma"]:
        r = subprocess.run([sys.executable, __file__, c], capture_output=True, text=True)
        print(c, "rc", r.returncode, (r.stdout + r.stderr).strip().splitlines()[-1:] )
    sys.exit(0)
import torch
from paper_2403_16526_b200 import ops, _capi
kind, path = case.split("_")
h = 8 if path == "tma" else 7
dims = (h, 5, 6); S, hd = 1, 6; n = h * 30
cfg = ops.AttentionConfig(S, hd, 3)
Q = torch.randn(S * hd, n, device="cuda"); K = torch.randn(S * hd, n, device="cuda")
B = torch.randn(S, 27, device="cuda")
SF, LSE = ops.modet_fwd(Q, K, B, dims, cfg, layout=1)
torch.cuda.synchronize()
if kind == "fwd":
    print("ok"); sys.exit(0)
g = torch.randn(3 * S, n, device="cuda")
L = _capi.lib()
gQ = torch.zeros_like(Q); gK = torch.zeros_like(K); gB = torch.zeros_like(B)
args = [Q.data_ptr(), K.data_ptr(), B.data_ptr(), SF.data_ptr(), LSE.data_ptr(), g.data_ptr(),
        ops.dims3(dims), S, hd, 3, 1]
if kind == "row":
    rc = L.mdg_modet_bwd(*args, gQ.data_ptr(), None, gB.data_ptr(), 0, None)
else:
    rc = L.mdg_modet_bwd(*args, None, gK.data_ptr(), None, 0, None)
torch.cuda.synchronize()
print("ok rc", rc, L.mdg_last_error())
