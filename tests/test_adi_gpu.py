"""ADI step on the GPU (partitioned NTDM + tiled transpose) against the same
step with the oracle as the solver."""

import numpy as np
import pytest
import torch

from paper_1804_09666_b200.adi import ADIStep

from test_adi_dist import CpuBackend, problem

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [256, 1000])
def test_adi_gpu_matches_oracle_step(cuda, n):
    xs, rhs, ys = problem(n)
    ref, _, _ = ADIStep(xs, ys, backend=CpuBackend())(rhs)
    step = ADIStep([a.to(cuda) for a in xs], [a.to(cuda) for a in ys])
    u, stx, sty = step(rhs.to(cuda))
    assert int(stx.sum()) == 0 and int(sty.sum()) == 0
    u = u.cpu().numpy()
    err = np.max(np.abs(u - ref.numpy())) / np.max(np.abs(ref.numpy()))
    assert err <= 1e-12


def test_transpose_kernel(cuda):
    from paper_1804_09666_b200.adi import CudaBackend
    a = torch.randn(1000, 333, dtype=torch.float64, device=cuda)
    b = torch.empty(333, 1000, dtype=torch.float64, device=cuda)
    CudaBackend(cuda).transpose(a, b)
    assert torch.equal(b, a.t())
