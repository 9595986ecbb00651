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
