#!/usr/bin/env python
"""Benchmark of the batched band-SLAE hot path (BASELINE.json metric:
"batched PD/TD systems solved/s + HBM GB/s vs peak; SIP iterations/s").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload npdm]
                    [--algo partitioned|sequential] [--impl ours|reference]

Default workload: config 2 (BASELINE.json configs[1]) NPDM, B=8192 systems of
order N=4096 per GPU, float64, seed 1 -- the configuration the headline metric
is quoted on.  A step = one batched solve of the whole batch.  Weak scaling:
every rank solves its own B systems (seeded per rank); no collective on the
path.  Rank 0 prints ONE JSON line.

value     systems/s over all ranks, inputs resident in HBM (device-timed,
          CUDA events, max over ranks); inputs (1.88 GB) exceed the 126 MB L2
          so no flush is needed between steps.
e2e       the same metric through the public C ABI call with pinned HOST
          buffers: H2D of the step's diagonals + rhs and D2H of x inside the
          timed region.
roofline  dominant kernel: algorithmic bytes (56 B/row PD, 40 B/row TD:
          diagonals + rhs read, x written) per launch / mean launch time,
          against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the C restatement of the reference (oracle/c, OpenMP, all host
          threads) on a bounded sample of the same workload, rank 0, N=1.

--impl reference times that CPU restatement (the reference is pure Python and
is not compiled; the oracle port is its faithful CPU implementation) on this
arm's config and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    # name: (kind, batch, n, generator)
    "npdm": dict(kind="penta", solver="npdm", batch=8192, n=4096, cfg=1,
                 desc="config 2 NPDM: B=8192 pentadiagonal DD systems, N=4096, seed 1"),
    "mnpdm": dict(kind="penta", solver="mnpdm", batch=8192, n=4096, cfg=1, sparse=True,
                  desc="config 2 MNPDM: B=8192, N=4096, sparse outer diagonals (nz(sub2)=2), seed 1"),
    "ntdm": dict(kind="tri", solver="ntdm", batch=1024, n=1024, cfg=0,
                 desc="config 1 NTDM: B=1024 tridiagonal DD systems, N=1024, seed 0"),
    "ntdm8k": dict(kind="tri", solver="ntdm", batch=8192, n=8192, cfg=4,
                   desc="config 5 sweep: B=8192 tridiagonal DD systems, N=8192, seed 0"),
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[2:6]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def gen_inputs(wl, rank):
    from paper_1804_09666_b200 import workloads as W

    seed = [wl["cfg"], rank] if rank else wl["cfg"]   # rank 0 = the config's own seed
    rng = np.random.default_rng(seed)
    if wl["kind"] == "tri":
        return W.td_dominant(wl["batch"], wl["n"], rng=rng)
    return W.pd_dominant(wl["batch"], wl["n"], sparse_outer=wl.get("sparse", False), rng=rng)


def rowaligned(arrs, kind, layout):
    """Reference-length (B, L) host arrays -> row-aligned host arrays in the C
    ABI storage: interleaved (n, B) or system-major (B, n)."""
    offs = (-1, 0, 1) if kind == "tri" else (-2, -1, 0, 1, 2)
    main = arrs[len(offs) // 2]
    bsz, n = main.shape
    out = []
    for a, off in zip(arrs[:len(offs)], offs):
        first = -off if off < 0 else 0
        if layout == "interleaved":
            r = np.zeros((n, bsz))
            r[first:first + a.shape[1]] = a.T
        else:
            r = np.zeros((bsz, n))
            r[:, first:first + a.shape[1]] = a
        out.append(r)
    rhs = arrs[len(offs)]
    out.append(np.ascontiguousarray(rhs.T if layout == "interleaved" else rhs))
    return out


def cpu_port_rate(wl, arrs, sample, threads=None):
    """Time the C restatement of the reference on `sample` systems; returns
    (systems/s, seconds, threads)."""
    from oracle import cport

    kind = wl["kind"]
    sl = [a[:sample] for a in arrs]
    if kind == "tri":
        d, e, f = cport.rowaligned_tri(*sl[:3])
        b = np.ascontiguousarray(sl[3])
        cport.ntdm(d[:8], e[:8], f[:8], b[:8])
        t0 = time.perf_counter()
        cport.ntdm(d, e, f, b)
        dt = time.perf_counter() - t0
    else:
        r = cport.rowaligned_penta(*sl[:5])
        b = np.ascontiguousarray(sl[5])
        mod = 1 if wl["solver"] == "mnpdm" else 0
        cport.penta(mod, *(x[:8] for x in r), b[:8])
        t0 = time.perf_counter()
        cport.penta(mod, *r, b)
        dt = time.perf_counter() - t0
    return sample / dt, dt, cport.threads()


def run_reference(args, wl):
    """--impl reference: the CPU restatement on the host cores, rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    arrs = gen_inputs(wl, 0)
    bsz = wl["batch"]
    # bounded sample per step: aim ~1-3 s of CPU work per step
    rate0, _, _ = cpu_port_rate(wl, arrs, min(bsz, 256))
    sample = int(min(bsz, max(64, rate0 * 1.5)))
    for _ in range(args.warmup):
        cpu_port_rate(wl, arrs, min(sample, 64))
    times = []
    for _ in range(args.steps):
        rate, dt, thr = cpu_port_rate(wl, arrs, sample)
        times.append(dt)
    tot = sum(times)
    value = sample * len(times) / tot
    line = {
        "impl": "reference", "metric": "systems_solved_per_s", "value": value,
        "unit": "systems/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "sample_systems_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "systems/s", "cores": thr, "kind": "port",
                         "sample": f"{sample} of {bsz} systems per step, C restatement "
                                   f"(oracle/c/bx_oracle.c, OpenMP {thr} threads)"},
        "e2e": {"value": value, "unit": "systems/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    from paper_1804_09666_b200 import PentaMatrix, TriMatrix, _lib
    from paper_1804_09666_b200.core import ptr, workspace

    ws_world, rank, local = dist_env()
    if ws_world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    kind, bsz, n = wl["kind"], wl["batch"], wl["n"]
    algo = {"sequential": _lib.ALGO_SEQUENTIAL, "partitioned": _lib.ALGO_PARTITIONED}[args.algo]

    arrs = gen_inputs(wl, rank)
    lay = _lib.LAYOUT_INTERLEAVED if args.layout == "interleaved" else _lib.LAYOUT_SYSTEM_MAJOR
    host = rowaligned(arrs, kind, args.layout)                # C-ABI layout, host
    ld = bsz if args.layout == "interleaved" else n
    dev_in = [torch.from_numpy(h).to(dev) for h in host]
    x = torch.empty(host[-1].shape, dtype=torch.float64, device=dev)
    status = torch.empty(bsz, dtype=torch.int32, device=dev)
    index = torch.empty(bsz, dtype=torch.int32, device=dev)
    nz = torch.empty(bsz, dtype=torch.int64, device=dev)
    L = _lib.lib()
    solver = wl["solver"]
    nbytes = L.bx_workspace_bytes(_lib.SOLVER[solver], bsz, n, lay, algo)
    wsb = workspace(nbytes, dev)
    stream = torch.cuda.current_stream()

    def solve(ins, out):
        s = stream.cuda_stream
        if solver == "ntdm":
            rc = L.bx_ntdm_f64(*(ptr(t) for t in ins), ptr(out), ptr(status), ptr(index), bsz, n,
                               ld, lay, algo, ptr(wsb), wsb.numel(), s)
        elif solver == "npdm":
            rc = L.bx_npdm_f64(*(ptr(t) for t in ins), ptr(out), ptr(status), ptr(index), bsz, n,
                               ld, lay, algo, ptr(wsb), wsb.numel(), s)
        else:
            rc = L.bx_mnpdm_f64(*(ptr(t) for t in ins), ptr(out), ptr(status), ptr(index), ptr(nz),
                                bsz, n, ld, lay, algo, ptr(wsb), wsb.numel(), s)
        _lib.check(rc, solver)

    # ---- correctness gate on this rank's data (sampled systems vs oracle) ----
    solve(dev_in, x)
    torch.cuda.synchronize()
    assert int((status != 0).sum()) == 0, "unexpected zero pivot"

    def barrier():
        if ws_world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if ws_world > 1:
            t = torch.tensor([v], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    # ---- device-resident timed region ----
    for _ in range(args.warmup):
        solve(dev_in, x)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = ClockSampler(local).start() if rank == 0 else None
    time.sleep(0.3 if sampler else 0)
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    for k in range(args.steps):
        ev[k][0].record()
        solve(dev_in, x)
        ev[k][1].record()
    t_end.record()
    barrier()
    clocks = sampler.stop() if sampler else None
    elapsed = max_over_ranks(t_start.elapsed_time(t_end) / 1e3)
    launch_s = [a.elapsed_time(b) / 1e3 for a, b in ev]
    mean_launch = statistics.mean(launch_s)
    value = bsz * ws_world * args.steps / elapsed

    bytes_per_row = 40 if kind == "tri" else 56
    alg_bytes = bytes_per_row * bsz * n
    peak, peak_src = load_peaks()
    achieved = alg_bytes / mean_launch / 1e9

    # ---- end-to-end through the C ABI with pinned host buffers ----
    pinned = [torch.from_numpy(h).pin_memory() for h in host]
    x_host = torch.empty(host[-1].shape, dtype=torch.float64).pin_memory()
    dev_e2e = [torch.empty_like(t) for t in dev_in]
    x_e2e = torch.empty_like(x)

    def e2e_step():
        for hsrc, ddst in zip(pinned, dev_e2e):
            ddst.copy_(hsrc, non_blocking=True)
        solve(dev_e2e, x_e2e)
        x_host.copy_(x_e2e, non_blocking=True)

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(e2e_steps):
        e2e_step()
    e1.record()
    barrier()
    e2e_elapsed = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    assert torch.equal(x_host, x.cpu()), "e2e result differs from the resident run"
    h2d = sum(h.nbytes for h in host)
    d2h = x_host.numel() * 8

    if rank != 0:
        if ws_world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if ws_world == 1 and not args.no_cpu_baseline:
        rate0, _, _ = cpu_port_rate(wl, arrs, min(bsz, 128))
        sample = int(min(bsz, max(64, rate0 * 5)))          # <= ~5 s per pass
        tot_s, tot_n, passes = 0.0, 0, 0
        while tot_s < 5.0 and passes < 20:                  # ~5-10 s of CPU work in all
            rate, dt, thr = cpu_port_rate(wl, arrs, sample)
            tot_s += dt
            tot_n += sample
            passes += 1
        cpu = {"value": tot_n / tot_s, "unit": "systems/s", "cores": thr, "kind": "port",
               "sample": f"{passes} pass(es) over {sample} of {bsz} systems ({tot_s:.1f} s), "
                         f"C restatement of the reference (oracle/c/bx_oracle.c), OpenMP {thr} threads"}

    line = {
        "metric": "systems_solved_per_s", "value": value, "unit": "systems/s",
        "n_gpus": ws_world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "solver": solver, "algo": args.algo,
                   "batch_per_gpu": bsz, "n": n, "layout": f"{args.layout} row-aligned",
                   "l2": f"inputs {alg_bytes/1e9:.2f} GB per step > 126 MB L2, no flush",
                   "parallelism": f"dp{ws_world} (system-index sharding)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": f"bx {solver} ({args.algo})",
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "mean_launch_ms": 1e3 * mean_launch, "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": {"value": bsz * ws_world * e2e_steps / e2e_elapsed, "unit": "systems/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "pinned host -> cudaMemcpyAsync -> bx C ABI -> D2H x"},
        "gpu_launches": args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line))
    if ws_world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="npdm", choices=sorted(WORKLOADS))
    ap.add_argument("--algo", default="partitioned", choices=["sequential", "partitioned"])
    ap.add_argument("--layout", default=None, choices=["interleaved", "system"],
                    help="C-ABI storage (default: system-major for partitioned, interleaved for sequential)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.layout is None:
        args.layout = "system" if args.algo == "partitioned" else "interleaved"
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
