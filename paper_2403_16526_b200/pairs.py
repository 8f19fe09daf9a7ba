"""Pair-parallel batch registration.

Every pairwise optimisation fine-tunes its own copy of the parameters
(engine.hpp:377-411), so a batch of pairs shards with no data-path collective:
pair i runs on rank i mod world, each rank on its own GPU, and only the final
per-pair results are gathered (one `all_gather_object`).  The reference runs
the batch one pair after another in a single process (cli.cpp:231).

    results = run_pairs(64, lambda i: register_pair(*load(i)))

`register_pair` is the per-pair unit on the native model driver; `run_pairs`
is the host-side sharding and gather, covered over gloo by tests/test_pairs.py.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import torch
import torch.distributed as dist


def shard(n_pairs: int, world: int, rank: int) -> List[int]:
    """Round-robin assignment: the pair indices rank `rank` owns."""
    if n_pairs < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError(f"shard: bad (n_pairs={n_pairs}, world={world}, rank={rank})")
    return list(range(rank, n_pairs, world))


def _world(group) -> tuple:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def run_pairs(n_pairs: int, register: Callable[[int], dict], group=None) -> List[dict]:
    """Runs `register(i)` for this rank's pairs, then gathers every rank's
    results; returns the list for all `n_pairs` in pair order on every rank.
    Each result is a dict; "pair" is set to its index."""
    world, rank = _world(group)
    mine = []
    for i in shard(n_pairs, world, rank):
        # a failing pair must not leave the other ranks blocked in the gather:
        # its error travels with the results and is re-raised on every rank
        try:
            r = dict(register(i))
        except Exception as e:  # noqa: BLE001
            if world == 1:
                raise
            r = {"error": f"{type(e).__name__}: {e}"}
        r["pair"] = i
        mine.append(r)
    if world == 1:
        return mine
    parts: List[Optional[list]] = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    out = sorted((r for p in parts for r in p), key=lambda r: r["pair"])
    errs = [r for r in out if "error" in r]
    if errs:
        raise RuntimeError("run_pairs: " + "; ".join(f"pair {r['pair']}: {r['error']}"
                                                       for r in errs))
    if [r["pair"] for r in out] != list(range(n_pairs)):
        raise RuntimeError("run_pairs: gathered results do not cover every pair once")
    return out


def register_pair(fixed, moving, params, iters=50, lr=1e-4, labels_fixed=None,
                  labels_moving=None, loss=None, keep_phi=False) -> dict:
    """One pairwise optimisation on the current GPU through the native model
    driver (mdg_model_*).  `params` are the 75 initial tensors (copied, so one
    initialisation serves every pair).  Returns the loss trace, the Dice trace
    when labels are given, and optionally the final deformation."""
    from . import ops

    dev = fixed.device
    model = ops.NativeModel([t.to(dev, copy=True) for t in params], tuple(fixed.shape[::-1][:3]),
                            loss=loss)
    trace, dice, phi = model.pairwise_optimize(fixed, moving, iters=iters, lr=lr,
                                               labels_fixed=labels_fixed,
                                               labels_moving=labels_moving)
    out = {"loss_trace": trace, "final_loss": trace[-1]}
    if dice:
        out["dice_trace"] = dice
        out["final_dice"] = dice[-1]
    if keep_phi:
        out["phi"] = phi.cpu()
    return out
