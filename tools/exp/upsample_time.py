"""upsample2 fwd / bwd device time at the pyramid's level shapes (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_16526_b200 import ops  # noqa: E402


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


for coarse in ((80, 96, 112), (40, 48, 56), (20, 24, 28), (10, 12, 14)):
    fine = tuple(2 * v for v in coarse)
    x = torch.randn(3, coarse[2], coarse[1], coarse[0], device="cuda")
    g = torch.randn(3, fine[2], fine[1], fine[0], device="cuda")
    gi = torch.zeros_like(x)
    f_us = t(lambda: ops.upsample_field_2x(x, fine, coarse))
    b_us = t(lambda: ops.upsample_field_2x_bwd(g, coarse, fine, gin=gi))
    print(f"coarse {coarse}: fwd {f_us:.1f} us, bwd {b_us:.1f} us")
