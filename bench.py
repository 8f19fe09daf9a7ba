#!/usr/bin/env python
"""bench.py — ModeT hot-path benchmark (B200, sm_100a).

Workload (BASELINE.json north_star unit): the finest pyramid level L1 of the
small preset at 160x192x224 — ModeT operator forward + backward (S=1 head,
d=6) plus the trilinear feature warp forward + backward (C=8 channels).
One "step" = modet_fwd + modet_bwd + warp_fwd + warp_bwd over one volume whose
synthetic inputs (seeded, the reference bench's distributions) are already
resident in HBM.  The step footprint (~1.4 GB) is far larger than L2
(126 MB), so no explicit flush is needed between steps.

Metric: Gvoxel/s of that step (voxels processed / second, whole job).  With
N ranks (torchrun, one GPU each) every rank processes its own independent
volume (pair-parallel, no data-path collective): weak scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every key.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = (160, 192, 224)  # h, w, l  (x, y, z)
S, HD, NB, CH = 1, 6, 3, 8
LAYOUT = 1  # MDG_QK_PLANAR: the fused tier's native {S*d, n} layout
METRIC = "ModeT op fwd+bwd + feature warp fwd+bwd throughput at 160x192x224 (L1, S=1, d=6, C=8)"
UNIT = "Gvoxel/s"

# SURVEY.md §8(d) algorithmic bytes per voxel (fp32, each tensor once per
# direction, W never materialised)
BYTES = {
    "modet_fwd": 4 * (2 * S * HD + 3 * S),
    "modet_bwd": 4 * (4 * S * HD + 3 * S),
    "warp_fwd": 4 * (3 + 2 * CH),
    "warp_bwd": 4 * (6 + 3 * CH),
}
KERNEL_NAMES = {  # op -> the CUDA kernels it launches (ncu names, in launch order)
    "modet_fwd": ["modet_fwd_tiled_k", "modet_fwd_fixup_k"],
    "modet_bwd": ["modet_bwd_row_k", "modet_bwd_col_k", "reduce_db_k"],
    "warp_fwd": ["warp_fwd_k"],
    "warp_bwd": ["warp_bwd_k"],
}


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_ncu_traffic():
    """dram bytes per launch of each kernel, from the committed ncu --set full
    capture of this bench's step (profiles/ncu_traffic.json, written by
    profiles/summarize_ncu.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def op_traffic(op):
    """ncu DRAM bytes of one launch of `op` (sum over its kernels), or None
    when the committed capture lacks one of them."""
    t = load_ncu_traffic().get("kernels", {})
    vals = [t.get(k, {}).get("dram_bytes") for k in KERNEL_NAMES[op]]
    vals = [v for k, v in zip(KERNEL_NAMES[op], vals) if v is not None or k in t]
    if not vals or any(v is None for v in vals):
        return None
    return int(sum(vals))


# ------------------------------------------------------------ clock sampler
class ClockSampler:
    """Polls NVML while the timed region runs (SM clock, max clock, reasons)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        reasons = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ our arm
def make_inputs(rank: int):
    """Seeded synthetic inputs (bench.cpp:28-35 distributions): Q, K ~ U(-1,1),
    B ~ U(-0.5,0.5); upstream gSF ~ U(-1,1); features ~ N(0,1); a smooth-ish
    displacement field of up to ~2 voxels; warp upstream gradient ~ N(0,1).
    Rank r uses seeds offset by r (independent pairs)."""
    import torch

    from paper_2403_16526_b200 import ops

    h, w, l = DIMS
    n = h * w * l
    base = 1000 * rank
    r = ops.Rng(5 + base)
    # drawn in the reference's position-major order, stored planar {S*d, n}
    Q = r.uniform((n, S * HD), -1.0, 1.0).t().contiguous()
    K = r.uniform((n, S * HD), -1.0, 1.0).t().contiguous()
    B = r.uniform((S, 27), -0.5, 0.5)
    gSF = ops.Rng(6 + base).uniform((3 * S, n), -1.0, 1.0)
    feat = ops.Rng(7 + base).normal((CH, l, w, h))
    # phi = make_smooth_velocity(dims, seed 11, 2.0 vox, sigma 4)
    # (synth.cpp:75-90, native and bit-identical)
    field = ops.make_smooth_velocity(DIMS, 11 + base, 2.0, 4.0)
    gout = ops.Rng(9 + base).normal((CH, l, w, h))
    return dict(Q=Q, K=K, B=B, gSF=gSF, feat=feat, field=field, gout=gout)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2403_16526_b200 import _capi, ops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _capi.lib()
    assert L.mdg_device_ok() == 1, "libmdg needs an sm_100a device"

    h, w, l = DIMS
    n = h * w * l
    cfg = ops.AttentionConfig(S, HD, NB)
    host_in = make_inputs(rank)
    d_in = {k: v.to(dev) for k, v in host_in.items()}
    Q, K, B, gSF = d_in["Q"], d_in["K"], d_in["B"], d_in["gSF"]
    feat, field, gout = d_in["feat"], d_in["field"], d_in["gout"]
    SF = torch.empty(3 * S, n, device=dev)
    LSE = torch.empty(S, n, device=dev)
    gQ, gK, gB = torch.zeros_like(Q), torch.zeros_like(K), torch.zeros_like(B)
    warped = torch.empty_like(feat)
    gin, gfield = torch.zeros_like(feat), torch.zeros_like(field)
    d3 = ops.dims3(DIMS)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream

    def chk(rc):
        if rc != 0:
            raise RuntimeError(L.mdg_last_error().decode())

    ops_order = ["modet_fwd", "modet_bwd", "warp_fwd", "warp_bwd"]

    def step(ev=None):
        # forward outputs are overwritten; the ModeT backward writes fresh
        # gQ/gK (accumulate=0, as for a tape's zero-initialised grads); the
        # warp backward accumulates (reference contract)
        if ev: ev[0].record(st)
        chk(L.mdg_modet_fwd(Q.data_ptr(), K.data_ptr(), B.data_ptr(), d3, S, HD, NB, LAYOUT,
                            SF.data_ptr(), LSE.data_ptr(), None, sp))
        if ev: ev[1].record(st)
        chk(L.mdg_modet_bwd(Q.data_ptr(), K.data_ptr(), B.data_ptr(), SF.data_ptr(),
                            LSE.data_ptr(), gSF.data_ptr(), d3, S, HD, NB, LAYOUT,
                            gQ.data_ptr(), gK.data_ptr(), gB.data_ptr(), 0, sp))
        if ev: ev[2].record(st)
        chk(L.mdg_warp_fwd(feat.data_ptr(), CH, d3, field.data_ptr(), warped.data_ptr(), sp))
        if ev: ev[3].record(st)
        chk(L.mdg_warp_bwd(feat.data_ptr(), CH, d3, field.data_ptr(), gout.data_ptr(),
                           gin.data_ptr(), gfield.data_ptr(), sp))
        if ev: ev[4].record(st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    K_ = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K_)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.mdg_launch_count()
    with ClockSampler(local) as clk:
        t0.record(st)
        for i in range(K_):
            step(evs[i])
        t1.record(st)
        torch.cuda.synchronize()
    launches = L.mdg_launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / K_
    per_op = {op: statistics.mean(evs[i][j].elapsed_time(evs[i][j + 1]) for i in range(K_))
              for j, op in enumerate(ops_order)}
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * n / (ms_max * 1e-3) / 1e9

    # ---------------- e2e: the reference-facing host-buffer C-ABI calls
    e2e = None if args.no_e2e else run_e2e(args, L, host_in, world, dev)

    # ---------------- the decoding pyramid around the op,
    # reported beside the headline (it is not part of `value`)
    pyramid = None if args.no_pyramid else run_pyramid(dev)
    po = None if args.no_po else run_po(dev, world, args.po_pairs)

    # the warp's worst case for gather locality: i.i.d. random_field (test_util.hpp:40-48)
    warp_rf = None if args.no_random_field else run_warp_random_field(L, d3, feat, gout, rank,
                                                                     dev, st)
    # config 2: the registration forward at 160x192x160 (LPBA-shaped)
    cfg2 = None if args.no_cfg2 else run_cfg2(dev)

    peak, peak_kind = load_peak()
    stress = None if args.no_stress else run_modet_stress(L, rank, dev, st, peak)
    slab_po_res = None if args.no_slab_po else run_slab_po(dev, world)
    dom = max(per_op, key=lambda k: per_op[k])
    achieved = BYTES[dom] * n / (per_op[dom] * 1e-3) / 1e9
    traffic = op_traffic(dom)
    step_bytes = sum(BYTES.values()) * n
    result = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": K_, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Rng streams, bench.cpp distributions)",
        "config": {"workload": "L1 160x192x224: ModeT fwd+bwd (S=1,d=6,nb=3) + warp fwd+bwd (C=8)",
                   "dims": list(DIMS), "heads": S, "head_dim": HD, "channels": CH,
                   "parallelism": f"pair-parallel x{world} (independent volume per GPU)",
                   "l2": "inputs larger than L2 (step footprint ~1.4 GB), no flush"},
        "per_op_ms": {k: round(v, 4) for k, v in per_op.items()},
        "roofline": {"bound": "hbm", "op": dom, "kernel": " + ".join(KERNEL_NAMES[dom]),
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full of this step)",
                     "peak_kind": peak_kind,
                     "bytes_per_launch": BYTES[dom] * n},
        "roofline_per_op": {op: {"ms": round(per_op[op], 4), "alg_bytes": BYTES[op] * n,
                                 "frac": round(BYTES[op] * n / (per_op[op] * 1e-3) / 1e9 / peak, 4),
                                 "ncu_dram_bytes": op_traffic(op)} for op in ops_order},
        "roofline_step": {"achieved": round(step_bytes / (ms_max * 1e-3) / 1e9, 1),
                          "peak": peak, "unit": "GB/s",
                          "frac": round(step_bytes / (ms_max * 1e-3) / 1e9 / peak, 4),
                          "bytes_per_step": step_bytes},
        "e2e": e2e,
        "warp_random_field": warp_rf,
        "modet_stress": stress,
        "slab_po": slab_po_res,
        "cfg2": cfg2,
        "pyramid": pyramid,
        "po": po,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_warp_random_field(L, d3, feat, gout, rank, dev, st, reps=10):
    """Warp fwd + bwd (C=8) at 160x192x224 with the i.i.d. random_field
    displacement (|phi| in [0.3, 2] voxels, random sign per entry): the gather
    / scatter locality worst case, timed beside the smooth-field headline."""
    import torch

    from paper_2403_16526_b200 import ops

    fld = ops.random_field(DIMS, 12 + 1000 * rank, 2.0).to(dev)
    out = torch.empty_like(feat)
    gin, gf = torch.zeros_like(feat), torch.zeros_like(fld)
    sp = st.cuda_stream

    def go(ev=None):
        if ev: ev[0].record(st)
        L.mdg_warp_fwd(feat.data_ptr(), CH, d3, fld.data_ptr(), out.data_ptr(), sp)
        if ev: ev[1].record(st)
        L.mdg_warp_bwd(feat.data_ptr(), CH, d3, fld.data_ptr(), gout.data_ptr(), gin.data_ptr(),
                       gf.data_ptr(), sp)
        if ev: ev[2].record(st)

    for _ in range(3):
        go()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    for e in evs:
        go(e)
    torch.cuda.synchronize()
    n = DIMS[0] * DIMS[1] * DIMS[2]
    f = statistics.median(e[0].elapsed_time(e[1]) for e in evs)
    b = statistics.median(e[1].elapsed_time(e[2]) for e in evs)
    return {"field": "random_field(dims, seed 12, mag 2.0) (test_util.hpp:40-48)",
            "warp_fwd_ms": round(f, 4), "warp_bwd_ms": round(b, 4),
            "Gvoxel_per_s": round(n / ((f + b) * 1e-3) / 1e9, 3)}


def run_modet_stress(L, rank, dev, st, peak, reps=5):
    """SURVEY §8(d) op-at-scale stress: the ModeT operator fwd + bwd with
    S = 8 heads of d = 8 at 160x192x224 (Q, K {64, n}: 1.76 GB each), the
    bench.cpp distributions, device-resident; timed beside the headline."""
    import torch

    from paper_2403_16526_b200 import ops

    S8, D8 = 8, 8
    n = DIMS[0] * DIMS[1] * DIMS[2]
    g = torch.Generator(device=dev).manual_seed(77 + rank)
    Q = torch.rand(S8 * D8, n, device=dev, generator=g) * 2 - 1
    K = torch.rand(S8 * D8, n, device=dev, generator=g) * 2 - 1
    B = torch.rand(S8, 27, device=dev, generator=g) - 0.5
    gSF = torch.rand(3 * S8, n, device=dev, generator=g) * 2 - 1
    SF = torch.empty(3 * S8, n, device=dev)
    LSE = torch.empty(S8, n, device=dev)
    gQ, gK, gB = torch.empty_like(Q), torch.empty_like(K), torch.zeros_like(B)
    d3 = ops.dims3(DIMS)
    sp = st.cuda_stream
    P = lambda t: t.data_ptr()  # noqa: E731

    def go(ev=None):
        if ev: ev[0].record(st)
        rc = L.mdg_modet_fwd(P(Q), P(K), P(B), d3, S8, D8, NB, LAYOUT, P(SF), P(LSE), None, sp)
        if ev: ev[1].record(st)
        rc |= L.mdg_modet_bwd(P(Q), P(K), P(B), P(SF), P(LSE), P(gSF), d3, S8, D8, NB, LAYOUT,
                              P(gQ), P(gK), P(gB), 0, sp)
        if ev: ev[2].record(st)
        if rc:
            raise RuntimeError(L.mdg_last_error().decode())

    for _ in range(2):
        go()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    for e in evs:
        go(e)
    torch.cuda.synchronize()
    f = statistics.median(e[0].elapsed_time(e[1]) for e in evs)
    b = statistics.median(e[1].elapsed_time(e[2]) for e in evs)
    fwd_bytes, bwd_bytes = 4 * (2 * S8 * D8 + 3 * S8) * n, 4 * (4 * S8 * D8 + 3 * S8) * n
    return {"workload": "ModeT fwd+bwd, S=8, d=8, nb=3 at 160x192x224 (SURVEY 8d stress)",
            "fwd_ms": round(f, 4), "bwd_ms": round(b, 4),
            "Gvoxel_per_s": round(n / ((f + b) * 1e-3) / 1e9, 3),
            "frac_fwd": round(fwd_bytes / (f * 1e-3) / 1e9 / peak, 4),
            "frac_bwd": round(bwd_bytes / (b * 1e-3) / 1e9 / peak, 4),
            "alg_bytes_fwd_bwd": fwd_bytes + bwd_bytes}


def run_cfg2(dev, reps=5):
    """BASELINE config 2: the registration forward (encoder x2 -> 5-level
    ModeT pyramid with RegHead and warps -> NCC/grad_reg loss) of the small
    preset on the synthetic LPBA-shaped pair make_synth_pair(160x192x160,
    seed 1), init_model(42) weights, native driver; device time per forward."""
    import torch

    from paper_2403_16526_b200 import ops

    dims = (160, 192, 160)
    f, m, _, _, _ = ops.synth_pair(dims, seed=1, max_disp=2.0)
    f, m = f.to(dev), m.to(dev)
    model = ops.NativeModel([t.to(dev) for t in ops.init_model(42)], dims)
    for _ in range(2):
        model.loss_step(f, m, backward=False)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        e[0].record()
        model.loss_step(f, m, backward=False)
        e[1].record()
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    ms = statistics.median(ts)
    del model
    return {"workload": "registration forward (encoder x2 + 5-level pyramid + loss), small "
                        "preset, make_synth_pair(160x192x160, seed 1)",
            "fwd_ms": round(ms, 3), "pairs_per_sec_forward_only": round(1e3 / ms, 2)}


def run_pyramid(dev, reps=5):
    """Decoder pyramid (build_pipeline minus the encoder, small preset: heads
    8,4,2,1,1, hd 6, channels 128..8) on synthetic features at 160x192x224:
    device time of one forward and one backward (CUDA events)."""
    import torch

    from paper_2403_16526_b200 import ops

    dims = [DIMS]
    for _ in range(4):
        dims.append(tuple((v + 1) // 2 for v in dims[-1]))
    dims = dims[::-1]
    chans, heads = (128, 64, 32, 16, 8), (8, 4, 2, 1, 1)
    g = torch.Generator(device=dev).manual_seed(0)
    ff = [torch.randn(c, d[2], d[1], d[0], device=dev, generator=g) for c, d in zip(chans, dims)]
    mf = [torch.randn(c, d[2], d[1], d[0], device=dev, generator=g) for c, d in zip(chans, dims)]
    lps = []
    for c, Sh in zip(chans, heads):
        K = Sh * HD
        lps.append(ops.LevelParams(
            ops.ProjectionParams(torch.randn(K, c, device=dev, generator=g) * 0.3,
                                 torch.zeros(K, device=dev), torch.ones(K, device=dev),
                                 torch.zeros(K, device=dev)),
            torch.randn(Sh, 27, device=dev, generator=g) * 0.5,
            torch.randn(3, 3 * Sh, 3, 3, 3, device=dev, generator=g) * 0.01,
            torch.zeros(3, device=dev)))
    cfg = ops.ModelConfig(heads_per_level=heads, head_dim=HD)
    pyr = ops.Pyramid(cfg, dims, chans, check_finite=False)
    gphi = torch.randn(3, DIMS[2], DIMS[1], DIMS[0], device=dev, generator=g)
    grads = [p.zeros_like() for p in lps]
    gf = [torch.zeros_like(t) for t in ff]
    gm = [torch.zeros_like(t) for t in mf]
    for _ in range(2):
        pyr.forward(ff, mf, lps)
        pyr.backward(gphi, grads, gf, gm)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(reps):
        e[0].record()
        pyr.forward(ff, mf, lps)
        e[1].record()
        pyr.backward(gphi, grads, gf, gm)
        e[2].record()
        torch.cuda.synchronize()
        tf.append(e[0].elapsed_time(e[1]))
        tb.append(e[1].elapsed_time(e[2]))
    # one decoder PO iteration (engine.hpp:377-411 minus the encoder): pyramid
    # forward -> loss (NCC + grad_reg on the full-resolution images) -> loss
    # backward -> pyramid backward -> Adam over every decoder parameter
    fixed = torch.rand(1, DIMS[2], DIMS[1], DIMS[0], device=dev, generator=g)
    moving = torch.rand(1, DIMS[2], DIMS[1], DIMS[0], device=dev, generator=g)
    params = [t for lp in lps for t in lp.tensors()]
    opt = ops.AdamOptimizer(params)
    lcfg = ops.LossConfig(lam=1.0, ncc_window=9)

    def po_iter():
        for gr in grads:
            for t in gr.tensors():
                t.zero_()
        phi = pyr.forward(ff, mf, lps)
        ops.total_loss(fixed, moving, phi, lcfg)
        gphi_ = ops.total_loss_bwd(fixed, moving, phi, lcfg)[0]
        pyr.backward(gphi_, grads, gf, gm)
        opt.step(1e-4, [t for gr in grads for t in gr.tensors()])

    po_iter()
    torch.cuda.synchronize()
    tp = []
    for _ in range(reps):
        e[0].record()
        po_iter()
        e[1].record()
        torch.cuda.synchronize()
        tp.append(e[0].elapsed_time(e[1]))
    return {"workload": "decoder pyramid (build_pipeline minus encoder), small preset, "
                        "160x192x224 fine level, synthetic features",
            "fwd_ms": round(statistics.median(tf), 3), "bwd_ms": round(statistics.median(tb), 3),
            "decoder_iter_ms": round(statistics.median(tp), 3),
            "decoder_iter_note": "pyramid fwd + NCC/grad_reg loss fwd+bwd + pyramid bwd + "
                                 "Adam with the encoder features held fixed (the full "
                                 "iteration is under 'po')",
            "arena_mib": round(pyr.device_bytes / 2 ** 20, 1)}


def run_slab_po(dev, world, reps=3, reach=6):
    """BASELINE config 3: the PO iteration of one 160x192x224 pair split along z
    over the ranks (paper_2403_16526_b200/slab_po.py: halo exchange and
    all-reduces over the job's process group, NCCL).  Device time of `reps`
    iterations between barriers, max over ranks; at N = 1 also the fixed-reach
    step replayed as one CUDA graph.  Strong scaling: the pair is fixed."""
    import torch

    from paper_2403_16526_b200 import ops, slab_po

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return round(float(t.item()), 3)

    try:
        params = [t.to(dev) for t in ops.init_model(42)]
        f, m, _, _, _ = ops.synth_pair(DIMS, seed=1, max_disp=2.0)
        model = slab_po.SlabModel(params, DIMS, reach=reach)
        fl, ml = model.local(f.to(dev)), model.local(m.to(dev))
        # eager with a fixed reach (no host round trip inside the step; the
        # host-side floor of an eager step is ~15.6 ms, tools/exp/slab_cpu_floor.py)
        out = {"workload": "PO iteration of one 160x192x224 pair over z-slabs (config 3)",
               "slab_depths": [b - a for a, b in slab_po.split_units(DIMS[2], world)],
               "scaling": "strong", "reach_planes": reach,
               "eager_ms_per_iter": timed(lambda: model.po_step(fl, ml))}
        if world == 1:  # (multi-rank capture of the NCCL exchange is not exercised here)
            g = slab_po.SlabModel(params, DIMS, reach=reach)
            out["graph_ms_per_iter"] = timed(lambda: g.po_step(fl, ml, graph=True))
        return out
    except Exception as e:  # reported, never fatal for the headline line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def run_po(dev, world, pairs=0, reps=5):
    """Pairwise optimisation (engine.hpp:377-411) of the full small-preset
    model at 160x192x224: ms per PO iteration (encoder x2 -> pyramid -> NCC +
    grad_reg -> backward -> Adam), and pairs/sec for 50-iteration pairs
    (50 iterations + the final evaluation forward).  `pairs` > 0 runs that many
    complete pairs and times them; otherwise pairs/sec is derived from the
    measured iteration and forward times (labelled)."""
    import torch

    from paper_2403_16526_b200 import ops

    params = [t.to(dev) for t in ops.init_model(42)]
    model = ops.NativeModel(params, DIMS)  # mdg_model_*: the C++ model driver
    # make_synth_pair(dims, seed, max_disp 2.0), native, bit-identical
    fixed, moving, _, _, _ = ops.synth_pair(DIMS, seed=1, max_disp=2.0)
    fixed, moving = fixed.to(dev), moving.to(dev)
    # a dedicated stream: the legacy default stream cannot be captured, and the
    # iteration runs as one CUDA graph (mdg_model_po_step)
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream())
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ti, tf = [], []
    with torch.cuda.stream(side):
        for _ in range(3):  # eager, capture, replay
            model.po_step(fixed, moving)
        torch.cuda.synchronize()
        for _ in range(reps):
            e[0].record()
            model.po_step(fixed, moving)
            e[1].record()
            model.loss_step(fixed, moving, backward=False)
            e[2].record()
            torch.cuda.synchronize()
            ti.append(e[0].elapsed_time(e[1]))
            tf.append(e[1].elapsed_time(e[2]))
    it_ms, fwd_ms = statistics.median(ti), statistics.median(tf)
    if world > 1:  # the slowest rank sets the pair rate
        import torch.distributed as dist

        t = torch.tensor([it_ms, fwd_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        it_ms, fwd_ms = float(t[0].item()), float(t[1].item())
    out = {"workload": "PO of the small-preset model at 160x192x224 (make_synth_pair seed 1, "
                       "init_model(42) weights), native model driver (mdg_model_*), "
                       "one CUDA graph per iteration",
           "iter_ms": round(it_ms, 3), "final_forward_ms": round(fwd_ms, 3),
           "iters_per_pair": 50,
           "pairs_per_sec": round(world * 1e3 / (50 * it_ms + fwd_ms), 4),
           "pairs_per_sec_kind": "derived: world / (50 x iter + final forward), timed on the device"}
    if pairs > 0:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(side):
            for _ in range(pairs):
                m = ops.NativeModel([t.to(dev) for t in ops.init_model(42)], DIMS)
                for _ in range(50):
                    m.po_step(fixed, moving)
                m.loss_step(fixed, moving, backward=False)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if world > 1:  # the slowest rank sets the pair rate
            import torch.distributed as dist

            tw = torch.tensor([wall], device=dev, dtype=torch.float64)
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
            wall = float(tw.item())
        out["pairs_run"] = pairs
        out["pairs_per_sec_measured"] = round(world * pairs / wall, 4)
        out["pairs_per_sec_measured_kind"] = ("wall clock per rank (init_model + model setup + "
                                              "50 graph-replayed updates + final forward)")
    return out


def run_e2e(args, L, host_in, world, dev):
    """Same metric through the host-buffer drop-ins (mdg_*_host): pinned host
    inputs in, host outputs back, copies inside the timed region.  Same
    semantics as the device step: the ModeT backward overwrites gQ/gK/gB
    (accumulate=0), the warp backward accumulates (the reference's rule)."""
    import torch

    from paper_2403_16526_b200 import ops

    h, w, l = DIMS
    n = h * w * l
    pin = {k: v.pin_memory() for k, v in host_in.items()}
    outs = {
        "SF": torch.empty(3 * S, n).pin_memory(), "LSE": torch.empty(S, n).pin_memory(),
        "gQ": torch.zeros(n, S * HD).pin_memory(), "gK": torch.zeros(n, S * HD).pin_memory(),
        "gB": torch.zeros(S, 27).pin_memory(), "warped": torch.empty(CH, l, w, h).pin_memory(),
        "gin": torch.zeros(CH, l, w, h).pin_memory(), "gfield": torch.zeros(3, l, w, h).pin_memory(),
    }
    d3 = ops.dims3(DIMS)
    p = lambda t: t.data_ptr()  # noqa: E731

    def step():
        rc = L.mdg_modet_fwd_host(p(pin["Q"]), p(pin["K"]), p(pin["B"]), d3, S, HD, NB, LAYOUT,
                                  p(outs["SF"]), p(outs["LSE"]))
        rc |= L.mdg_modet_bwd_host(p(pin["Q"]), p(pin["K"]), p(pin["B"]), p(outs["SF"]),
                                   p(outs["LSE"]), p(pin["gSF"]), d3, S, HD, NB, LAYOUT,
                                   p(outs["gQ"]), p(outs["gK"]), p(outs["gB"]), 0)
        rc |= L.mdg_warp_fwd_host(p(pin["feat"]), CH, d3, p(pin["field"]), p(outs["warped"]))
        rc |= L.mdg_warp_bwd_host(p(pin["feat"]), CH, d3, p(pin["field"]), p(pin["gout"]),
                                  p(outs["gin"]), p(outs["gfield"]))
        if rc:
            raise RuntimeError(L.mdg_last_error().decode())

    step()
    steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    t0 = time.perf_counter()
    per_step = []
    for _ in range(steps):
        ts = time.perf_counter()
        step()
        per_step.append((time.perf_counter() - ts) * 1e3)
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([dt], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    f4 = 4
    # bytes the calls move over PCIe (counted from the tensors they copy); the
    # gradient accumulators stay on the host (host-side += of the device
    # contribution), so they cross only once, device -> host
    h2d = (2 * n * S * HD + 27 * S) * f4 \
        + (2 * n * S * HD + 27 * S + 3 * n * S + n * S + 3 * n * S + 27 * S) * f4 \
        + (CH * n + 3 * n) * f4 + (2 * CH * n + 3 * n) * f4
    d2h = (4 * n * S) * f4 + (2 * n * S * HD + 27 * S) * f4 + CH * n * f4 + (CH * n + 3 * n) * f4
    return {"value": round(world * n / dt / 1e9, 5), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 3),
            "ms_steps": [round(x, 2) for x in per_step],
            "api": "mdg_modet_fwd_host + mdg_modet_bwd_host + mdg_warp_fwd_host + "
                   "mdg_warp_bwd_host (pinned host buffers)", "steps": steps}


# ----------------------------------------------------- reference CPU arm
REF_SLAB_Z = 32  # each worker's bounded sample: a 160x192x32 depth slab (W alone
                 # is 106 MB per worker: not cache-resident; 2 of 32 planes are
                 # slab boundaries)


def _ref_worker_inputs(seed):
    import pyoracle

    h, w, _ = DIMS
    dims = (h, w, REF_SLAB_Z)
    n = h * w * REF_SLAB_Z
    r = pyoracle.Rng(seed)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    Q = f(r.uniform(n * S * HD, -1, 1).reshape(n, S * HD))
    K = f(r.uniform(n * S * HD, -1, 1).reshape(n, S * HD))
    B = f(r.uniform(S * 27, -0.5, 0.5).reshape(S, 27))
    gSF = f(pyoracle.Rng(seed + 1).uniform(3 * S * n, -1, 1).reshape(3 * S, REF_SLAB_Z, w, h))
    feat = f(pyoracle.Rng(seed + 2).normal(CH * n).reshape(CH, REF_SLAB_Z, w, h))
    # the same field distribution as the GPU arm: make_smooth_velocity (synth.cpp:75-90)
    fld = f(pyoracle.ref().make_smooth_velocity(dims, seed + 3, 2.0, 4.0))
    gout = f(pyoracle.Rng(seed + 4).normal(CH * n).reshape(CH, REF_SLAB_Z, w, h))
    return dims, (Q, K, B, gSF, feat, fld, gout)


def _ref_step(lib, dims, inp):
    """The reference's own hot path (attention.hpp + sampling.hpp kernels as
    op_na_fused / op_subfields / op_warp call them), one slab."""
    Q, K, B, gSF, feat, fld, gout = inp
    W, err = lib.na_fwd(Q, K, B, dims, S, HD, NB)
    assert err is None
    lib.subfields_fwd(W, dims, S, NB)
    gW = lib.subfields_bwd(gSF, dims, S, NB)
    lib.na_bwd(Q, K, W, gW, dims, S, HD, NB)
    lib.warp_fwd(feat, fld)
    lib.warp_bwd(feat, fld, gout)


def _cpu_run(kind, threads, steps, warmup):
    """Run `threads` workers in parallel (ctypes releases the GIL), each on
    its own slab; returns (Gvoxel/s, seconds per step, voxels per step)."""
    import pyoracle

    if kind == "reference":
        lib = pyoracle.ref_fast()  # -O3, native ISA
    else:
        lib = pyoracle.mdo()
    work = [_ref_worker_inputs(100 + 17 * i) for i in range(threads)]
    nvox = sum(d[0] * d[1] * d[2] for d, _ in work)

    def one_step():
        ts = [threading.Thread(target=_ref_step, args=(lib, d, inp)) for d, inp in work]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    for _ in range(warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    dt = (time.perf_counter() - t0) / max(steps, 1)
    return nvox / dt / 1e9, dt, nvox


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(seconds):
    """Reference CPU path (oracle/_ref, compiled from the reference sources)
    on the host cores, bounded to ~`seconds` of work."""
    import pyoracle

    kind = "reference" if pyoracle.ref_available() else "port"
    threads = cpu_threads()
    v, dt, nvox = _cpu_run(kind, threads, 1, 0)
    steps = max(1, int(seconds / max(dt, 1e-3)) - 1)
    if steps > 1:
        v, dt, nvox = _cpu_run(kind, threads, steps, 0)
    return {"value": round(v, 6), "unit": UNIT, "cores": threads, "kind": kind,
            "build": os.path.basename(pyoracle.ref_fast_path()) if kind == "reference" else "mdo",
            "sample": f"{threads} threads x one 160x192x{REF_SLAB_Z} slab each "
                      f"({nvox} voxels/step), {steps} step(s) of {dt:.2f}s: "
                      "na_fused_fwd+subfields_fwd+subfields_bwd+na_fused_bwd+warp_fwd+warp_bwd",
            "ms_per_step": round(dt * 1e3, 1)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import pyoracle

    kind = "reference" if pyoracle.ref_available() else "port"
    threads = cpu_threads()
    v, dt, nvox = _cpu_run(kind, threads, args.steps, args.warmup)
    out = {
        "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Rng streams)",
        "config": {"workload": "L1 160x192x224: ModeT fwd+bwd (S=1,d=6,nb=3) + warp fwd+bwd (C=8)",
                   "sample": f"per step: {threads} CPU threads, one 160x192x{REF_SLAB_Z} slab each"},
        "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": threads, "kind": kind,
                         "build": os.path.basename(pyoracle.ref_fast_path()),
                         "sample": f"{threads} x 160x192x{REF_SLAB_Z} slabs ({nvox} voxels) per step"},
        "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling)")
    ap.add_argument("--no-pyramid", action="store_true", help="skip the pyramid timing")
    ap.add_argument("--no-po", action="store_true", help="skip the PO-iteration timing")
    ap.add_argument("--no-slab-po", action="store_true",
                    help="skip the depth-slab PO (config 3) timing")
    ap.add_argument("--no-stress", action="store_true",
                    help="skip the S=8, d=8 ModeT stress timing")
    ap.add_argument("--no-random-field", action="store_true",
                    help="skip the random_field warp timing")
    ap.add_argument("--no-cfg2", action="store_true", help="skip the config-2 forward timing")
    ap.add_argument("--po-pairs", type=int, default=1,
                    help="run this many complete 50-iteration pairs (pairs/sec measured, "
                         "wall clock: model setup + 50 updates + the final evaluation)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        run_reference(args)
    else:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        run_ours(args)


if __name__ == "__main__":
    main()
