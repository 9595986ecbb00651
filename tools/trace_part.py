"""Developer tool: per-phase clocks of the partitioned kernel (trace build).

Builds a -DBX_TRACE variant of libbandix_b200 under /tmp, runs one solve and
prints the median cycles spent per phase.  Not used by the product or bench."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1804_09666_b200 import build as B  # noqa: E402

out = "/tmp/bxtrace"
os.makedirs(out, exist_ok=True)
objs = []
for src in B.sources():
    o = os.path.join(out, os.path.basename(src) + ".o")
    subprocess.run([B.nvcc(), *B.ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", B.INCLUDE,
                    "-I", B.CSRC, "-DBX_TRACE",
                    "-DBX_TRACE_BASE=" + os.environ.get("BX_TRACE_BASE", "0"), "-c", src, "-o", o], check=True)
    objs.append(o)
lib = os.path.join(out, "libbxtrace.so")
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"], check=True)
from paper_1804_09666_b200 import _lib  # noqa: E402
_lib.LIB_PATH = lib
L = _lib.lib()
L.bx_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
dev = torch.device("cuda", 0)
arrs = [torch.rand((batch, n), dtype=torch.float64, device=dev) - 0.5 for _ in range(2 * k + 2)]
arrs[k] += 4.0
x = torch.empty((batch, n), dtype=torch.float64, device=dev)
st = torch.empty(batch, dtype=torch.int32, device=dev)
ix = torch.empty(batch, dtype=torch.int32, device=dev)
p = lambda t: t.data_ptr()  # noqa: E731
s = torch.cuda.current_stream().cuda_stream
nws = L.bx_workspace_bytes(0 if k == 1 else 1, batch, n, 1, 1)
ws = torch.empty(nws, dtype=torch.uint8, device=dev)
for _ in range(3):
    if k == 1:
        rc = L.bx_ntdm_f64(*(p(a) for a in arrs), p(x), p(st), p(ix), batch, n, n, 1, 1, p(ws), nws, s)
    else:
        rc = L.bx_npdm_f64(*(p(a) for a in arrs), p(x), p(st), p(ix), batch, n, n, 1, 1, p(ws), nws, s)
    assert rc == 0, L.bx_last_error()
torch.cuda.synchronize()
buf = np.zeros((4096, 24), dtype=np.int64)
L.bx_trace_read(buf.ctypes.data, buf.nbytes)
names = ["down", "up", "port+warp-asc", "xwarp-asc", "cluster", "descent", "phase3", "status"]
d = np.diff(buf[:, :9], axis=1)
ok = buf[:, 0] > 0
print(f"K={k} n={n} B={batch} cfg={os.environ.get('BX_PART_CFG', 'auto')} CTAs traced={ok.sum()}")
for j, nm in enumerate(names):
    print(f"  {nm:10s} median {np.median(d[ok, j]):9.0f} cyc   p90 {np.percentile(d[ok, j], 90):9.0f}")
for nm, a, b in (("clu:lane0", 4, 12), ("clu:syncwarp", 12, 5), ("desc:xwarp", 5, 10), ("xw:offs", 5, 13), ("xw:levels", 13, 15), ("xw:wlr", 15, 10), ("desc:sync", 10, 11), ("desc:inwarp", 11, 6)):
    dd = buf[ok, b] - buf[ok, a]
    print(f"  {nm:10s} median {np.median(dd):9.0f} cyc   p90 {np.percentile(dd, 90):9.0f}")
tot = buf[ok, 8] - buf[ok, 0]
print(f"  total      median {np.median(tot):9.0f} cyc   p90 {np.percentile(tot, 90):9.0f}")
# per-SM occupancy of the memory phase: fraction of the traced window during
# which at least one resident CTA of that SM is in its down (load) pass
fr = []
for sm in np.unique(buf[ok, 9]):
    sel = ok & (buf[:, 9] == sm)
    iv = sorted(zip(buf[sel, 0], buf[sel, 1]))
    lo, hi = buf[sel, 0].min(), buf[sel, 8].max()
    cov, cs, ce = 0, None, None
    for a, b in iv:
        if cs is None or a > ce:
            if cs is not None:
                cov += ce - cs
            cs, ce = a, b
        else:
            ce = max(ce, b)
    cov += ce - cs
    fr.append(cov / max(1, hi - lo))
print(f"  SMs {len(fr)}: down-pass coverage median {np.median(fr):.2f}  "
      f"CTAs/SM median {np.median(np.bincount(buf[ok, 9].astype(int))[np.unique(buf[ok, 9]).astype(int)]):.0f}")
