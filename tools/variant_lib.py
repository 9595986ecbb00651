"""Developer tool: build a variant of libbandix_b200 with extra nvcc flags
into a directory outside the package (for A/B sweeps), e.g.

    python tools/variant_lib.py /tmp/v1 -DBX_NLW2=1
    BX_LIB=/tmp/v1/libbandix_b200.so python tools/sweep_part.py child 2 4096 8192
"""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1804_09666_b200 import build as B  # noqa: E402

out, flags = sys.argv[1], sys.argv[2:]
os.makedirs(out, exist_ok=True)
objs, procs = [], []
for src in B.sources():
    o = os.path.join(out, os.path.basename(src) + ".o")
    procs.append(subprocess.Popen([B.nvcc(), *B.ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                                   "-I", B.INCLUDE, "-I", B.CSRC, "--expt-relaxed-constexpr", *flags,
                                   "-c", src, "-o", o]))
    objs.append(o)
assert all(p.wait() == 0 for p in procs)
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", os.path.join(out, "libbandix_b200.so"), *objs,
                "-lcudart"], check=True)
print(os.path.join(out, "libbandix_b200.so"))
