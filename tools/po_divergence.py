"""Where do the GPU and reference PO trajectories part?  (diagnostic)

At the initial parameters P0 of a 32^3 synth pair: per-tensor gradient error
and Adam-step sign disagreements between the GPU (ops.NativeModel) and the
reference run_loss_step; then, for each tensor i, the loss after one Adam step
with the reference's update everywhere except tensor i (the GPU's update
there), evaluated by the reference.  Prints the tensors whose GPU update moves
the loss the most.

    python tools/po_divergence.py [--perturbed]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import pyoracle  # noqa: E402
from paper_2403_16526_b200 import ops  # noqa: E402
from test_gpu_encoder import device_tensors, perturbed_model, split  # noqa: E402


def adam1(p, g, lr=1e-4, b1=0.9, b2=0.999, eps=1e-8):
    g = g.astype(np.float64)
    m = (1 - b1) * g
    v = (1 - b2) * g * g
    mh = m / (1 - b1)
    vh = v / (1 - b2)
    return (p - lr * mh / (np.sqrt(vh) + eps)).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--perturbed", action="store_true")
    ap.add_argument("--dims", type=int, default=32)
    ap.add_argument("--po", type=int, default=0, help="also compare N-iteration PO traces")
    a = ap.parse_args()
    ref = pyoracle.ref()
    dims = (a.dims,) * 3
    f, m, lf, lm, gt = ref.synth_pair(dims, seed=4, max_disp=2.0)
    if a.perturbed:
        packed, sizes = perturbed_model(ref, 6)
    else:
        packed, sizes = ref.model_params(42)
    loss_r, gp_r, _ = ref.loss_step(f, m, packed)
    nat = ops.NativeModel(device_tensors(packed, sizes), dims)
    terms, _ = nat.loss_step(torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda())
    torch.cuda.synchronize()
    g_g = [t.cpu().numpy().ravel() for t in nat.grads]
    g_r = split(gp_r, sizes)
    P0 = split(packed, sizes)
    print(f"loss gpu {float(terms[0]):.9g} ref {loss_r:.9g}")
    P1r = [adam1(p, g) for p, g in zip(P0, g_r)]
    P1g = [adam1(p, g) for p, g in zip(P0, g_g)]
    base, _, _ = ref.loss_step(f, m, np.concatenate(P1r), grads=False)
    allg, _, _ = ref.loss_step(f, m, np.concatenate(P1g), grads=False)
    print(f"loss after 1 Adam step: ref-update {base:.9g}  gpu-update {allg:.9g}  "
          f"rel {abs(allg - base) / abs(base):.3g}")
    rows = []
    for i in range(len(sizes)):
        flips = int(np.sum(np.sign(g_g[i]) != np.sign(g_r[i])))
        rn = float(np.linalg.norm(g_g[i] - g_r[i]) / max(np.linalg.norm(g_r[i]), 1e-30))
        hyb = list(P1r)
        hyb[i] = P1g[i]
        lh, _, _ = ref.loss_step(f, m, np.concatenate(hyb), grads=False)
        rows.append((abs(lh - base), i, sizes[i], flips, rn, float(np.abs(g_r[i]).max())))
    rows.sort(reverse=True)
    print("dloss      tensor size flips relnorm max|g_ref|")
    for r in rows[:20]:
        print(f"{r[0]:.3e} {r[1]:5d} {r[2]:6d} {r[3]:5d} {r[4]:.2e} {r[5]:.2e}")
    if a.po:
        lr_, dr_, _ = ref.pairwise_optimize(f, m, lf, lm, packed, a.po, lr=1e-4)
        nat2 = ops.NativeModel(device_tensors(packed, sizes), dims)
        lg_, dg_, _ = nat2.pairwise_optimize(
            torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda(), a.po, lr=1e-4,
            labels_fixed=torch.from_numpy(lf).cuda(), labels_moving=torch.from_numpy(lm).cuda())
        for i, (x, y, u, v) in enumerate(zip(lg_, lr_, dg_, dr_)):
            print(f"it {i:3d} loss {x:.7f} {y:.7f} rel {abs(x - y) / abs(y):.2e}  "
                  f"dice {u:.5f} {v:.5f} d {abs(u - v):.1e}")


if __name__ == "__main__":
    main()
