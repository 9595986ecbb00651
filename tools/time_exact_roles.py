"""Developer timing: the symbolic pivot pass alone (bx_det_band_f64 runs
exactly that pass) against the whole STDM / SPDM solve (pivot pass and
pivoted limit solve overlapped in one launch) on config-3 inputs.  Not part
of the product or the bench."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1804_09666_b200 import _lib, workloads as W
    from paper_1804_09666_b200.core import ptr, workspace
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    batch, n = 4096, 2048
    s = torch.cuda.current_stream().cuda_stream
    for kind in ("stdm", "spdm"):
        rng = np.random.default_rng(2)
        if kind == "stdm":
            sub, main_, sup, rhs, _ = W.td_symbolic(batch, n, rng=rng)
            diags = [None, sub, main_, sup, None]
            offs = (None, 1, 0, 0, None)
        else:
            s2, s1, main_, p1, p2, rhs, _ = W.pd_symbolic(batch, n, rng=rng)
            diags = [s2, s1, main_, p1, p2]
            offs = (2, 1, 0, 0, 0)
        # interleaved row-aligned: row i of system b at [i, b]; sub-diagonals
        # shifted to their row (lead zeros), super-diagonals padded at the end
        dev_d = []
        for d, o in zip(diags, offs):
            if d is None:
                dev_d.append(None)
                continue
            full = np.zeros((batch, n))
            if o:
                full[:, o:] = d
            else:
                full[:, :d.shape[1]] = d
            dev_d.append(torch.from_numpy(full.T.copy()).to(dev))
        b = torch.from_numpy(rhs.T.copy()).to(dev)
        x = torch.empty_like(b)
        st = torch.empty(batch, dtype=torch.int32, device=dev)
        subs = torch.empty(batch, dtype=torch.int32, device=dev)
        mant = torch.empty(batch, dtype=torch.float64, device=dev)
        expo = torch.empty(batch, dtype=torch.int64, device=dev)
        sid = _lib.SOLVER[kind]
        ws = workspace(L.bx_workspace_bytes(sid, batch, n, 0, 0), dev)
        P = lambda t: ptr(t) if t is not None else None  # noqa: E731

        def det():
            _lib.call("bx_det_band_f64", 1 if kind == "stdm" else 2, *(P(t) for t in dev_d),
                      ptr(mant), ptr(expo), ptr(st), None, ptr(subs), batch, n, batch, 0, s)

        def solve():
            if kind == "stdm":
                _lib.call("bx_stdm_f64", P(dev_d[1]), P(dev_d[2]), P(dev_d[3]), ptr(b), ptr(x),
                          ptr(st), None, ptr(subs), batch, n, batch, 0, ptr(ws), ws.numel(), s)
            else:
                _lib.call("bx_spdm_f64", *(P(t) for t in dev_d), ptr(b), ptr(x), ptr(st), None,
                          ptr(subs), batch, n, batch, 0, ptr(ws), ws.numel(), s)

        for name, fn in (("pivot pass (det_band)", det), ("whole solve", solve)):
            for _ in range(2):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                fn()
            e1.record()
            torch.cuda.synchronize()
            print(f"{kind} {name:24s} {e0.elapsed_time(e1) / 5:.3f} ms  subs[0]={int(subs[0])} st={int(st.abs().sum())}")


if __name__ == "__main__":
    main()
