import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import pyoracle
from _util import random_feature_map, random_field
from paper_2403_16526_b200 import ops
m = pyoracle.mdo()
for C in (1, 2, 3, 4, 8):
    d = (7, 6, 5)
    vol = random_feature_map(C, d, 3); fld = random_field(d, 4, 1.5)
    ref = m.warp_fwd(vol, fld)
    got = ops.warp(torch.from_numpy(vol).cuda(), torch.from_numpy(fld).cuda()).cpu().numpy()
    diff = np.abs(got - ref)
    print("C", C, "max", diff.max(), "per-ch mismatches", [(int((got[c] != ref[c]).sum())) for c in range(C)])
    go = random_feature_map(C, d, 5)
    gin, gf = ops.warp_bwd(torch.from_numpy(vol).cuda(), torch.from_numpy(fld).cuda(), torch.from_numpy(go).cuda())
    rgin, rgf = m.warp_bwd(vol, fld, go)
    print("   bwd gfield mism", int((gf.cpu().numpy() != rgf).sum()), "gin maxdiff", float(np.abs(gin.cpu().numpy() - rgin).max()))
