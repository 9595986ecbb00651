"""Developer sweep: partitioned-solver throughput across CTA configurations
and system orders (same total rows).  Not part of the product or the bench."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run_one(k, n, batch, steps=10):
    from paper_1804_09666_b200 import _lib
    from paper_1804_09666_b200.core import ptr, workspace
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    arrs = [torch.rand((batch, n), dtype=torch.float64, device=dev, generator=g) - 0.5 for _ in range(2 * k + 2)]
    arrs[k] += 4.0     # diagonal dominance
    x = torch.empty((batch, n), dtype=torch.float64, device=dev)
    st = torch.empty(batch, dtype=torch.int32, device=dev)
    ix = torch.empty(batch, dtype=torch.int32, device=dev)
    ws = workspace(L.bx_workspace_bytes(0 if k == 1 else 1, batch, n, 1, 1), dev)
    s = torch.cuda.current_stream().cuda_stream

    def go():
        if k == 1:
            rc = L.bx_ntdm_f64(*(ptr(a) for a in arrs), ptr(x), ptr(st), ptr(ix), batch, n, n, 1, 1, ptr(ws), ws.numel(), s)
        else:
            rc = L.bx_npdm_f64(*(ptr(a) for a in arrs), ptr(x), ptr(st), ptr(ix), batch, n, n, 1, 1, ptr(ws), ws.numel(), s)
        _lib.check(rc, "solve")
    for _ in range(3):
        go()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        go()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / steps / 1e3
    byts = (2 * k + 3) * 8 * n * batch
    return t, byts / t / 1e9


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        k, n, batch = map(int, sys.argv[2:5])
        t, gbs = run_one(k, n, batch)
        print(f"K={k} n={n:6d} B={batch:6d} cfg={os.environ.get('BX_PART_CFG','auto'):>4} {t*1e3:8.3f} ms {gbs:8.1f} GB/s")
        sys.exit(0)
    total = 8192 * 4096
    for k in (2, 1):
        for cfg in ["auto", "1", "2", "3", "4", "5", "6"]:
            for n in (1024, 2048, 4096, 8192):
                env = dict(os.environ)
                if cfg != "auto":
                    env["BX_PART_CFG"] = cfg
                else:
                    env.pop("BX_PART_CFG", None)
                r = subprocess.run([sys.executable, __file__, "child", str(k), str(n), str(total // n)],
                                   env=env, capture_output=True, text=True)
                print((r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:200], flush=True)
