"""System-index sharding on 2 gloo ranks (CPU): every rank solves its own
contiguous slice with the restatement; gathering the slices reproduces the
single-process solve bit for bit, and the MAX reduction of the residuals
equals the global maximum."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import direct as D
from paper_1804_09666_b200 import workloads as W
from paper_1804_09666_b200.sharding import gather_systems, global_max, shard_bounds, shard_rows


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = W.pd_dominant(37, 64, seed=5)                     # 37: uneven slices
    local, (lo, hi) = shard_rows(list(p), rank, world)
    x, st, _ = D.npdm(*local)
    res = D.residual_inf_penta(*local[:5], x, local[5])
    xg = gather_systems(torch.from_numpy(x), 37)
    rmax = global_max(torch.tensor([float(res.max())], dtype=torch.float64))
    if rank == 0:
        out.put((xg.numpy(), float(rmax[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_bounds_cover_batch():
    for batch in (0, 1, 7, 8, 37, 8192):
        for world in (1, 2, 3, 8):
            b = [shard_bounds(batch, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == batch
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


def test_two_rank_solve_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    xg, rmax = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = W.pd_dominant(37, 64, seed=5)
    x, _, _ = D.npdm(*p)
    assert np.array_equal(xg, x)
    assert rmax == float(D.residual_inf_penta(*p[:5], x, p[5]).max())
