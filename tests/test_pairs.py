"""Pair-parallel batch registration (paper_2403_16526_b200/pairs.py, SURVEY.md
§8(e) cfg5).  CPU: the round-robin shard and the result gather over gloo at
world sizes 2 and 3.  GPU: one pair through register_pair / run_pairs (the
native model driver, CUDA-graph iterations) against the reference
pairwise_optimize — the same Dice gate as test_gpu_encoder.py, which checks
the Python-composed driver."""
import json
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from _util import rel_norm
from paper_2403_16526_b200 import pairs


def test_shard_round_robin_covers_every_pair_once():
    for n in (0, 1, 5, 64):
        for world in (1, 2, 3, 8):
            owned = [pairs.shard(n, world, r) for r in range(world)]
            flat = sorted(i for o in owned for i in o)
            assert flat == list(range(n))
            for r, o in enumerate(owned):
                assert all(i % world == r for i in o)
    with pytest.raises(ValueError):
        pairs.shard(4, 2, 2)
    with pytest.raises(ValueError):
        pairs.shard(-1, 1, 0)


def test_run_pairs_single_process():
    out = pairs.run_pairs(4, lambda i: {"v": i * 10})
    assert [r["pair"] for r in out] == [0, 1, 2, 3]
    assert [r["v"] for r in out] == [0, 10, 20, 30]


def _worker(rank, world, port, n, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = pairs.run_pairs(n, lambda i: {"ran_on": rank, "v": i * i})
        with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
            json.dump(res, f)
    finally:
        dist.destroy_process_group()


def _failing_worker(rank, world, port, n, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def register(i):
        if i == 3:
            raise FloatingPointError("optimization: non-finite loss (nan)")
        return {"v": i}

    try:
        try:
            pairs.run_pairs(n, register)
            msg = "no error"
        except RuntimeError as e:
            msg = str(e)
        with open(os.path.join(out_dir, f"e{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,n", [(2, 7), (3, 5), (2, 1)])
def test_run_pairs_over_gloo(tmp_path, world, n):
    mp.start_processes(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    for res in got:  # every rank holds the full, ordered result list
        assert res == got[0]
        assert [r["pair"] for r in res] == list(range(n))
        for r in res:
            assert r["ran_on"] == r["pair"] % world
            assert r["v"] == r["pair"] ** 2


def test_run_pairs_failing_pair_raises_on_every_rank(tmp_path):
    """A pair that raises (e.g. NumericError on a non-finite loss) must not
    leave the other ranks blocked in the gather: every rank re-raises it."""
    world = 2
    mp.start_processes(_failing_worker, args=(world, _free_port(), 6, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    for r in range(world):
        msg = open(tmp_path / f"e{r}.txt").read()
        assert "pair 3" in msg and "non-finite loss" in msg, msg


@pytest.mark.gpu
def test_register_pair_native_dice_gate(cuda, ref, deterministic):
    """Two pairs through run_pairs / register_pair (the native model driver,
    one CUDA graph per iteration), 50 Adam iterations each, against the
    reference pairwise_optimize at every step."""
    from test_gpu_encoder import check_po_traces, device_tensors, reference_po

    dims, iters = (32, 32, 32), 50
    f, m, lf, lm, packed, sizes, loss_r, dice_r, phi_r = reference_po(ref, dims, iters)
    params = device_tensors(packed, sizes)
    fd, md = torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda()
    lfd, lmd = torch.from_numpy(lf).cuda(), torch.from_numpy(lm).cuda()
    out = pairs.run_pairs(2, lambda i: pairs.register_pair(
        fd, md, params, iters=iters, lr=1e-4, labels_fixed=lfd, labels_moving=lmd,
        keep_phi=True))
    assert [r["pair"] for r in out] == [0, 1]
    for r in out:
        assert len(r["loss_trace"]) == iters + 1 and len(r["dice_trace"]) == iters + 1
        check_po_traces(r["loss_trace"], r["dice_trace"], loss_r, dice_r)
        assert rel_norm(r["phi"].numpy(), phi_r) <= 1e-2
    # the initial parameters are copied: both pairs start from the same model
    # and (deterministic mode) the PO iteration is bit-reproducible, so the two
    # traces are identical
    assert out[0]["loss_trace"] == out[1]["loss_trace"], (out[0]["loss_trace"],
                                                          out[1]["loss_trace"])
