"""The ADI exchange (x-sweep -> all-to-all -> y-sweep) on 2 ranks over gloo,
with the oracle as the tridiagonal solver: the distributed step must equal
the single-process step bit-for-bit (the solves are identical per system;
only data movement differs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import direct as D
from paper_1804_09666_b200.adi import ADIStep
from paper_1804_09666_b200 import workloads as W


class CpuBackend:
    def tri_solve(self, sub1, main, sup1, rhs, out):
        x, st, _ = D.ntdm(sub1[:, 1:].numpy(), main.numpy(), sup1[:, :-1].numpy(), rhs.numpy())
        out.copy_(torch.from_numpy(x))
        return torch.from_numpy(st)

    def transpose(self, src, dst):
        dst.copy_(src.t())


def rowaligned(sub, main, sup):
    n = main.shape[1]
    s = np.zeros_like(main); s[:, 1:] = sub
    u = np.zeros_like(main); u[:, :n - 1] = sup
    return [torch.from_numpy(np.ascontiguousarray(a)) for a in (s, main, u)]


def problem(n):
    xs, ys = W.adi_step(n, seed=0)
    return rowaligned(*xs[:3]), torch.from_numpy(xs[3]), rowaligned(*ys)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, n, out, chunks):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    xs, rhs, ys = problem(n)
    ny_l, nx_l = n // world, n // world
    rows = slice(rank * ny_l, (rank + 1) * ny_l)
    cols = slice(rank * nx_l, (rank + 1) * nx_l)
    step = ADIStep([a[rows].contiguous() for a in xs], [a[cols].contiguous() for a in ys],
                   group=dist.group.WORLD, backend=CpuBackend(), chunks=chunks)
    u, _, _ = step(rhs[rows].contiguous())
    gathered = [torch.empty_like(u) for _ in range(world)]
    dist.all_gather(gathered, u)
    if rank == 0:
        out.put(torch.cat(gathered, 0).numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [1, 4, 5])
def test_adi_two_ranks_gloo_equals_single(chunks):
    # chunks > 1: the x-sweep runs in slices whose all-to-alls are queued
    # asynchronously (5 does not divide the 32 local rows: ragged slices)
    n = 64
    xs, rhs, ys = problem(n)
    single, _, _ = ADIStep(xs, ys, backend=CpuBackend())(rhs)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q, chunks)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, single.numpy())


def test_adi_step_matches_dense_solves():
    """x-sweep then y-sweep equals the two batches of direct solves."""
    n = 32
    xs, rhs, ys = problem(n)
    u, _, _ = ADIStep(xs, ys, backend=CpuBackend())(rhs)
    X = np.stack([np.linalg.solve(np.diag(xs[1][i].numpy()) + np.diag(xs[0][i, 1:].numpy(), -1)
                                  + np.diag(xs[2][i, :-1].numpy(), 1), rhs[i].numpy())
                  for i in range(n)])
    U = np.stack([np.linalg.solve(np.diag(ys[1][j].numpy()) + np.diag(ys[0][j, 1:].numpy(), -1)
                                  + np.diag(ys[2][j, :-1].numpy(), 1), X[:, j]) for j in range(n)])
    assert np.allclose(u.numpy(), U, rtol=1e-12, atol=1e-13)
