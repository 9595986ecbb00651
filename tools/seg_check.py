"""Developer check + sweep of the streaming partitioned solver (bx_direct_stream.cu):
parity of the partitioned path against the C restatement over many orders,
then device time per BX_SEG_CFG shape for config-2-sized batches.
Not part of the product or the bench."""
import os
import subprocess
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def parity():
    from oracle import cport
    from paper_1804_09666_b200 import PentaMatrix, TriMatrix, solve_npdm, solve_ntdm, solve_mnpdm
    from paper_1804_09666_b200 import workloads as W
    worst = 0.0
    for n in (4, 5, 8, 13, 100, 255, 256, 257, 1000, 1024, 1500, 2048, 3000, 4096, 5000, 8192, 12000, 16384):
        b = 16 if n > 4096 else 40
        p = W.pd_dominant(b, n, seed=n)
        ref, _, _, _ = cport.penta(0, *cport.rowaligned_penta(*p[:5]), np.ascontiguousarray(p[5]))
        A = PentaMatrix.from_diagonals(*p[:5], layout="system")
        r = solve_npdm(A, p[5], algo="partitioned", residual=False)
        x = r.x.cpu().numpy()
        e = float(np.max(np.abs(x - ref) / np.max(np.abs(ref), axis=1, keepdims=True)))
        st = r.status.cpu().numpy()
        rm = solve_mnpdm(A, p[5], algo="partitioned", residual=False)
        em = float(np.max(np.abs(rm.x.cpu().numpy() - ref) / np.max(np.abs(ref), axis=1, keepdims=True)))
        t = W.td_dominant(b, n, seed=n)
        reft, _, _ = cport.ntdm(*cport.rowaligned_tri(*t[:3]), np.ascontiguousarray(t[3]))
        T = TriMatrix.from_diagonals(*t[:3], layout="system")
        rt = solve_ntdm(T, t[3], algo="partitioned", residual=False)
        et = float(np.max(np.abs(rt.x.cpu().numpy() - reft) / np.max(np.abs(reft), axis=1, keepdims=True)))
        print(f"n={n:6d} penta err {e:.2e} mnpdm err {em:.2e} status {set(st.tolist())} | tri err {et:.2e} "
              f"status {set(rt.status.cpu().numpy().tolist())}", flush=True)
        worst = max(worst, e, em, et)
    # zero main diagonal at row 0: the reference raises ZeroPivot(0)
    p = W.pd_dominant(8, 4096, seed=5)
    p[2][3, 0] = 0.0
    A = PentaMatrix.from_diagonals(*p[:5], layout="system")
    r = solve_npdm(A, p[5], algo="partitioned", residual=False)
    print("zero pivot row 0: status", r.status.cpu().numpy().tolist(), "index", r.index.cpu().numpy().tolist())
    print("WORST", worst)


def timing(k, n, batch, steps=20):
    from paper_1804_09666_b200 import _lib
    from paper_1804_09666_b200.core import ptr, workspace
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    arrs = [torch.rand((batch, n), dtype=torch.float64, device=dev, generator=g) - 0.5 for _ in range(2 * k + 2)]
    arrs[k] += 4.0
    x = torch.empty((batch, n), dtype=torch.float64, device=dev)
    st = torch.empty(batch, dtype=torch.int32, device=dev)
    ix = torch.empty(batch, dtype=torch.int32, device=dev)
    solver = _lib.SOLVER["ntdm" if k == 1 else "npdm"]
    ws = workspace(L.bx_workspace_bytes(solver, batch, n, 1, 1), dev)
    s = torch.cuda.current_stream().cuda_stream

    def go():
        fn = L.bx_ntdm_f64 if k == 1 else L.bx_npdm_f64
        rc = fn(*(ptr(a) for a in arrs), ptr(x), ptr(st), ptr(ix), batch, n, n, 1, 1, ptr(ws), ws.numel(), s)
        _lib.check(rc, "solve")
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    assert int((st != 0).sum()) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        go()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / steps / 1e3
    byts = (2 * k + 3) * 8 * n * batch
    return t, byts / t / 1e9


if __name__ == "__main__":
    if sys.argv[1] == "parity":
        parity()
    elif sys.argv[1] == "child":
        k, n, batch = map(int, sys.argv[2:5])
        t, gbs = timing(k, n, batch)
        print(f"K={k} n={n:6d} B={batch:6d} cfg={os.environ.get('BX_SEG_CFG', 'auto'):>4} {t * 1e3:8.3f} ms "
              f"{gbs:8.1f} GB/s frac {gbs / 6545.9:.3f}", flush=True)
    else:
        total = 8192 * 4096
        cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto", "1", "2", "3", "6", "7"]
        ns = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [4096]
        for k in (2, 1):
            for n in ns:
                for cfg in cfgs:
                    env = dict(os.environ)
                    if cfg != "auto":
                        env["BX_SEG_CFG"] = cfg
                    else:
                        env.pop("BX_SEG_CFG", None)
                    r = subprocess.run([sys.executable, __file__, "child", str(k), str(n), str(total // n)],
                                       env=env, capture_output=True, text=True)
                    print((r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
