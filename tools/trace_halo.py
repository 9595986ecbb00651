"""Developer tool: per-phase clocks of the interface-iteration kernel
(bx_direct_halo.cu, -DBX_HALO_TRACE build under /tmp).  Runs one solve on
config-2-like data and prints the median cycles per phase of 4096 CTAs
starting at BX_HALO_TRACE_BASE.  Not used by the product or bench."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1804_09666_b200 import build as B  # noqa: E402

out = "/tmp/bxhalotrace"
os.makedirs(out, exist_ok=True)
objs, procs = [], []
extra = os.environ.get("BX_EXTRA_FLAGS", "").split()
for src in B.sources():
    o = os.path.join(out, os.path.basename(src) + ".o")
    procs.append(subprocess.Popen([B.nvcc(), *B.ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", B.INCLUDE,
                                   "-I", B.CSRC, "--expt-relaxed-constexpr", "-DBX_HALO_TRACE", *extra,
                                   "-DBX_HALO_TRACE_BASE=" + os.environ.get("BX_HALO_TRACE_BASE", "16384"),
                                   "-c", src, "-o", o]))
    objs.append(o)
assert all(p.wait() == 0 for p in procs)
lib = os.path.join(out, "libbxhalotrace.so")
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"], check=True)
from paper_1804_09666_b200 import _lib  # noqa: E402
_lib.LIB_PATH = lib
L = _lib.lib()
L.bx_halo_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
dev = torch.device("cuda", 0)
arrs = [torch.rand((batch, n), dtype=torch.float64, device=dev) * 2 - 1 for _ in range(2 * k + 2)]
arrs[k] = sum(a.abs() for i, a in enumerate(arrs[:2 * k + 1]) if i != k) + 1.0 + torch.rand_like(arrs[k])
x = torch.empty((batch, n), dtype=torch.float64, device=dev)
st = torch.empty(batch, dtype=torch.int32, device=dev)
ix = torch.empty(batch, dtype=torch.int32, device=dev)
p = lambda t: t.data_ptr()  # noqa: E731
s = torch.cuda.current_stream().cuda_stream
nws = L.bx_workspace_bytes(0 if k == 1 else 1, batch, n, 1, 1)
ws = torch.empty(nws, dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(4):
    if it == 3:
        e0.record()
    if k == 1:
        rc = L.bx_ntdm_f64(*(p(a) for a in arrs), p(x), p(st), p(ix), batch, n, n, 1, 1, p(ws), nws, s)
    else:
        rc = L.bx_npdm_f64(*(p(a) for a in arrs), p(x), p(st), p(ix), batch, n, n, 1, 1, p(ws), nws, s)
    assert rc == 0, L.bx_last_error()
e1.record()
torch.cuda.synchronize()
print(f"solve {e0.elapsed_time(e1):.3f} ms (trace build), retried systems: "
      f"{int(ws[4 * batch:8 * batch].view(torch.int32).sum())}")
buf = np.zeros((4096, 12), dtype=np.int64)
L.bx_halo_trace_read(buf.ctypes.data, buf.nbytes)
names = ["down", "up", "push+iface", "halo wait", "halo ifaces+sweeps", "phase3", "flags"]
d = np.diff(buf[:, :8], axis=1)
ok = buf[:, 0] > 0
print(f"K={k} n={n} B={batch} CTAs traced={ok.sum()}")
for j, nm in enumerate(names):
    print(f"  {nm:20s} median {np.median(d[ok, j]):9.0f} cyc   p90 {np.percentile(d[ok, j], 90):9.0f}")
tot = buf[ok, 7] - buf[ok, 0]
print(f"  total                median {np.median(tot):9.0f} cyc   p90 {np.percentile(tot, 90):9.0f}")
sms = buf[ok, 8].astype(int)
res = []
for sm in np.unique(sms):
    sel = ok & (buf[:, 8] == sm)
    lo, hi = buf[sel, 0].min(), buf[sel, 7].max()
    res.append(((buf[sel, 7] - buf[sel, 0]).sum() / max(1, hi - lo), sel.sum() * 1.0 / max(1, hi - lo)))
res = np.array(res)
print(f"  SMs {len(res)}: mean resident CTAs {np.median(res[:, 0]):.2f}, CTAs retired per Kcycle per SM {1e3 * np.median(res[:, 1]):.3f}")
