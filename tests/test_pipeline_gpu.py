"""Host-to-host pipelined solves (pipeline.py) equal the resident solve."""

import numpy as np
import pytest
import torch

from paper_1804_09666_b200.pipeline import HostPipeline
from paper_1804_09666_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("solver", ["ntdm", "npdm", "mnpdm"])
def test_pipeline_matches_oracle(cuda, solver):
    from oracle import cport
    B, n = 1000, 512
    if solver == "ntdm":
        d = W.td_dominant(B, n, seed=4)
        rows = list(cport.rowaligned_tri(*d[:3])) + [d[3]]
        ref, _, _ = cport.ntdm(*rows)
    else:
        d = W.pd_dominant(B, n, seed=4)
        rows = list(cport.rowaligned_penta(*d[:5])) + [d[5]]
        ref, _, _, _ = cport.penta(1 if solver == "mnpdm" else 0, *rows)
    pinned = [torch.from_numpy(np.ascontiguousarray(r)).pin_memory() for r in rows]
    xh = torch.empty((B, n), dtype=torch.float64).pin_memory()
    HostPipeline(solver, n, 128, cuda).run(pinned, xh)
    torch.cuda.synchronize()
    x = xh.numpy()
    assert np.max(np.abs(x - ref) / np.max(np.abs(ref), axis=1, keepdims=True)) <= 1e-10


def test_outer_lists_host_matches_device_compaction(cuda):
    """pipeline.outer_lists (host) == bx_outer_compact_f64 (device), and the
    sparse-outer pipeline reproduces the device solve."""
    import torch

    from paper_1804_09666_b200 import PentaMatrix, solve_mnpdm
    from paper_1804_09666_b200.pipeline import HostPipeline, outer_lists
    p = W.pd_dominant(24, 1500, seed=4, sparse_outer=True)
    A = PentaMatrix.from_diagonals(*p[:5], layout="system")
    S = A.sparse_outer()
    c, d, e, f, g = (t.cpu().numpy() for t in A.rowaligned())
    rows, vs, vp = outer_lists(c, g)
    assert np.array_equal(rows, S.rows.cpu().numpy())
    assert np.array_equal(vs, S.vals_sub2.cpu().numpy()) and np.array_equal(vp, S.vals_sup2.cpu().numpy())
    b = np.ascontiguousarray(p[5])
    host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (d, e, f, b)]
    lists = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (rows, vs, vp)]
    x = torch.empty((24, 1500), dtype=torch.float64).pin_memory()
    pipe = HostPipeline("mnpdm_sparse", 1500, 5, torch.device("cuda", 0), outer_k=rows.shape[1])
    pipe.run(host, x, host_outer=lists)
    torch.cuda.synchronize()
    ref = solve_mnpdm(S, p[5], algo="partitioned").x.cpu().numpy()
    assert np.array_equal(x.numpy(), ref)
