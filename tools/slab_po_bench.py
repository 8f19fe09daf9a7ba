"""Depth-slab PO benchmark (BASELINE config 3): one pair of 160x192x224
(make_synth_pair seed 1), the small preset, the PO iteration split along z
across the ranks (paper_2403_16526_b200/slab_po.py over NCCL).  Strong
scaling: the pair is fixed, each rank owns a slab.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \\
        --master-addr 127.0.0.1 --master-port P tools/slab_po_bench.py [--steps K]

Prints one JSON line from rank 0: ms per PO iteration (device time of K
iterations between barriers, max over ranks) and the single-volume native
driver's time for comparison at N = 1.  Modes: eager (data-dependent reach),
eager with a fixed reach, graph-replayed.  The graph mode at N > 1 captures
the NCCL exchange; it has only been run at N = 1 here (one GPU per call)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2403_16526_b200 import ops, slab_po  # noqa: E402

DIMS = (160, 192, 224)


def timed(fn, steps, dev, world):
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--reach", type=int, default=6,
                    help="fixed warp reach (planes) of the graph-replayed mode")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    params = [t.to(dev) for t in ops.init_model(42)]
    f, m, _, _, _ = ops.synth_pair(DIMS, seed=1, max_disp=2.0)
    model = slab_po.SlabModel(params, DIMS)
    fl, ml = model.local(f.to(dev)), model.local(m.to(dev))
    for _ in range(args.warmup):
        model.po_step(fl, ml)
    ms = timed(lambda: model.po_step(fl, ml), args.steps, dev, world)
    # fixed reach, eager: no host round trip inside the step (the host runs ahead)
    fmodel = slab_po.SlabModel(params, DIMS, reach=args.reach)
    for _ in range(args.warmup):
        fmodel.po_step(fl, ml)
    fms = timed(lambda: fmodel.po_step(fl, ml), args.steps, dev, world)
    # fixed reach: no host round trip inside the step, replayed as one CUDA graph
    gmodel = slab_po.SlabModel(params, DIMS, reach=args.reach)
    for _ in range(args.warmup):
        gmodel.po_step(fl, ml, graph=True)
    gms = timed(lambda: gmodel.po_step(fl, ml, graph=True), args.steps, dev, world)
    out = {"metric": "depth-slab PO iteration, small preset, 160x192x224 (config 3)",
           "ms_per_iter": round(ms, 3), "fixed_reach_eager_ms_per_iter": round(fms, 3),
           "graph_ms_per_iter": round(gms, 3),
           "graph_reach_planes": args.reach,
           "unit": "ms", "n_gpus": world, "scaling": "strong",
           "steps": args.steps, "slab_depths": [b - a for a, b in slab_po.split_units(DIMS[2],
                                                                                       world)]}
    if world == 1:
        nat = ops.NativeModel([t.to(dev) for t in ops.init_model(42)], DIMS)
        fd, md = f.to(dev), m.to(dev)
        for _ in range(args.warmup):
            nat.po_step(fd, md)
        out["native_graph_ms_per_iter"] = round(timed(lambda: nat.po_step(fd, md), args.steps,
                                                      dev, world), 3)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
