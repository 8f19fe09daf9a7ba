"""Depth-slab benchmark for BASELINE config 4: a CT-shaped 192x160x256 pair,
full-resolution ModeT (S=1, d=6) + feature warp (C=8) forward and backward,
the volume split along z across the ranks (paper_2403_16526_b200/slab.py:
halo planes over NCCL P2P, the warp's reach all-reduced).  Strong scaling:
the total volume is fixed, each rank owns one slab.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \\
        --master-addr 127.0.0.1 --master-port P tools/slab_bench.py [--steps K]

Prints one JSON line from rank 0: whole-volume Gvoxel/s over the device time
of K steps, max over ranks (CUDA events between barriers).  Verified here at
N = 1; the exchange itself is covered over gloo by tests/test_slab.py.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2403_16526_b200 import ops, slab as slabmod  # noqa: E402

DIMS = (192, 160, 256)  # h, w, l (x, y, z)
S, HD, CH = 1, 6, 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    h, w, l = DIMS
    sl = slabmod.Slab(h, w, l, world, rank)
    dz = sl.depth
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    mt = slabmod.SlabModeT(sl, S, HD)
    wp = slabmod.SlabWarp(sl)
    # the inputs written straight into the operator's extended buffers (no
    # staging copy; at N = 1 these are plain tensors)
    if world > 1:
        Q, K = mt.input_views(torch.empty(0, device=dev))
        gSF = mt.grad_view(torch.empty(0, device=dev))
    else:
        Q = torch.empty(S * HD, dz, w, h, device=dev)
        K = torch.empty_like(Q)
        gSF = torch.empty(3 * S, dz, w, h, device=dev)
    Q.copy_(torch.rand(S * HD, dz, w, h, device=dev, generator=g) * 2 - 1)
    K.copy_(torch.rand(S * HD, dz, w, h, device=dev, generator=g) * 2 - 1)
    B = torch.full((S, 27), 0.1, device=dev)
    gSF.copy_(torch.rand(3 * S, dz, w, h, device=dev, generator=g) * 2 - 1)
    feat = torch.randn(CH, dz, w, h, device=dev, generator=g)
    # a smooth displacement field of up to ~2 voxels (as the main bench):
    # random on a 16x coarser grid, trilinearly upsampled
    coarse = torch.rand(1, 3, max(2, dz // 16), max(2, w // 16), max(2, h // 16), device=dev,
                        generator=g) * 4 - 2
    field = torch.nn.functional.interpolate(coarse, size=(dz, w, h), mode="trilinear",
                                            align_corners=True)[0].contiguous()
    gout = torch.randn(CH, dz, w, h, device=dev, generator=g)

    def step():
        mt.forward(Q, K, B)
        mt.backward(gSF)
        wp.forward(feat, field)
        wp.backward(gout)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        n = h * w * l
        print(json.dumps({
            "metric": "depth-slab ModeT fwd+bwd + warp fwd+bwd throughput, 192x160x256 (config 4)",
            "value": round(n / (ms * 1e-3) / 1e9, 4), "unit": "Gvoxel/s", "n_gpus": world,
            "ms_per_step": round(ms, 4), "scaling": "strong", "steps": args.steps,
            "config": {"dims": list(DIMS), "heads": S, "head_dim": HD, "channels": CH,
                       "slab_depths": [b - a for a, b in slabmod.split(l, world)]}}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
