#!/usr/bin/env python
"""Benchmark of the batched band-SLAE hot path (BASELINE.json metric:
"batched PD/TD systems solved/s + HBM GB/s vs peak; SIP iterations/s").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload npdm]
                    [--algo partitioned|sequential] [--impl ours|reference]

Default workload: config 2 (BASELINE.json configs[1]) NPDM, B=8192 systems of
order N=4096 per GPU, float64, seed 1 -- the configuration the headline metric
is quoted on.  Other workloads (one JSON line each): mnpdm (config 2 sparse
outer), ntdm (config 1), ntdm8k (one config-5 sweep), sip (config 4:
512x512 grid, alpha 0.5; --sip-algo scan (default: correction form + row scans,
iteration count +-1) or wavefront (Algorithm 1 verbatim, bit parity)).

A step = one batched solve of the whole batch on every rank (weak scaling:
each rank its own seeded batch, no collective on the path).  Rank 0 prints
ONE JSON line.

value     the metric over all ranks, inputs resident in HBM (device-timed with
          CUDA events, max over ranks); inputs exceed the 126 MB L2 (config.l2).
e2e       the same metric through the C ABI with pinned HOST buffers: H2D of
          the step's matrix + rhs and D2H of x inside the timed region.
roofline  dominant kernel: algorithmic bytes per launch / mean launch time
          (CUDA events on the launching stream) vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the C restatement of the reference (oracle/c, OpenMP, all host
          threads) on a bounded sample of the same workload, rank 0, N=1.

--impl reference times that CPU restatement (the reference is pure Python and
is not compiled; the oracle port is its faithful CPU implementation).
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


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(args):
    """DRAM bytes per launch of the dominant kernel from the committed
    `ncu --set full` capture summary (profiles/traffic.json), if present."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            t = json.load(f)
        key = args.workload if args.workload != "npdm" or args.algo == "partitioned" else "npdm_seq"
        if args.workload == "sip" and args.sip_algo == "scan":
            key = "sip_scan"
        return t.get(key)
    except Exception:
        return None


def pcie_h2d_gbs(dev, nbytes=1 << 29, reps=3):
    """Pinned host -> device copy bandwidth on this box (the e2e ceiling)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index):
        self.gpu, self.rows, self.proc = gpu_index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
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


def rowaligned(arrs, offsets, layout):
    """Reference-length (B, L) host arrays + rhs -> row-aligned host arrays in
    the C ABI storage: interleaved (n, B) or system-major (B, n)."""
    main = arrs[offsets.index(0)]
    bsz, n = main.shape
    out = []
    for a, off in zip(arrs[:len(offsets)], offsets):
        first = -off if off < 0 else 0
        if layout == "interleaved":
            r = np.zeros((n, bsz)); r[first:first + a.shape[1]] = a.T
        else:
            r = np.zeros((bsz, n)); r[:, first:first + a.shape[1]] = a
        out.append(r)
    rhs = arrs[len(offsets)]
    out.append(np.ascontiguousarray(rhs.T if layout == "interleaved" else rhs))
    return out


DIRECT = {  # name: (solver, batch, n, config index, sparse outer, description)
    "npdm": ("npdm", 8192, 4096, 1, False,
             "config 2 NPDM: B=8192 pentadiagonal DD systems, N=4096, seed 1"),
    "mnpdm": ("mnpdm", 8192, 4096, 1, True,
              "config 2 MNPDM: B=8192, N=4096, sparse outer diagonals (nz(sub2)=2), seed 1"),
    "ntdm": ("ntdm", 1024, 1024, 0, False,
             "config 1 NTDM: B=1024 tridiagonal DD systems, N=1024, seed 0"),
    "ntdm8k": ("ntdm", 8192, 8192, 4, False,
               "config 5 sweep: B=8192 tridiagonal DD systems, N=8192"),
}


def direct_inputs(name, rank=0):
    from paper_1804_09666_b200 import workloads as W
    solver, bsz, n, cfg, sparse, _ = DIRECT[name]
    rng = np.random.default_rng([cfg, rank] if rank else cfg)
    if solver == "ntdm":
        return W.td_dominant(bsz, n, rng=rng)
    return W.pd_dominant(bsz, n, sparse_outer=sparse, rng=rng)


def cpu_direct_rate(solver, arrs, sample):
    """Time the C restatement on `sample` systems: (systems/s, seconds, threads)."""
    from oracle import cport
    sl = [a[:sample] for a in arrs]
    if solver == "ntdm":
        d, e, f = cport.rowaligned_tri(*sl[:3])
        b = np.ascontiguousarray(sl[3])
        cport.ntdm(d[:8], e[:8], f[:8], b[:8])
        t0 = time.perf_counter(); cport.ntdm(d, e, f, b); dt = time.perf_counter() - t0
    else:
        r = cport.rowaligned_penta(*sl[:5]); b = np.ascontiguousarray(sl[5])
        mod = 1 if solver == "mnpdm" else 0
        cport.penta(mod, *(x[:8] for x in r), b[:8])
        t0 = time.perf_counter(); cport.penta(mod, *r, b); dt = time.perf_counter() - t0
    return sample / dt, dt, cport.threads()


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def static_config(args, world):
    """The `config` object of the JSON line, identical for both arms (it depends
    on the command line only, never on the data or the device)."""
    w = args.workload
    par = (f"grid split over {world} ranks, NCCL all-to-all between sweeps" if w == "adi"
           else f"dp{world} (system-index sharding)")
    if w in DIRECT:
        solver, batch, n, cfg, sparse, desc = DIRECT[w]
        sparse = solver == "mnpdm" and sparse and args.algo == "partitioned"
        bpr = 40 if solver == "ntdm" or sparse else 56
        gb = bpr * batch * n / 1e9
        l2 = (f"inputs {gb:.2f} GB per step < 126 MB L2: L2 flushed (512 MB write) before every timed "
              "step; value and ms_per_step from the per-step CUDA events (flushes excluded)"
              if gb < 0.5 else f"inputs {gb:.2f} GB per step > 126 MB L2, no flush")
        c = {"workload": desc, "solver": solver, "algo": args.algo, "batch_per_gpu": batch, "n": n,
             "layout": f"{args.layout} row-aligned", "l2": l2}
        if sparse:
            c["outer"] = ("+-2 diagonals as per-system row lists, compacted once per matrix outside "
                          "the timed region")
    elif w == "sip":
        cs = SIP_CFG
        c = {"workload": (f"config 4 SIP: B={cs['batch']} five-point systems, {cs['n'] // cs['m']}x"
                          f"{cs['m']} grid (N={cs['n']}, offsets +-1, +-{cs['m']}), Stone alpha="
                          f"{cs['alpha']}, rel. tol 1e-8, <=500 iterations, seed {cs['cfg']}; a step = "
                          "one full sip_solve (ILU(0) + all iterations)"),
             "solver": "sip", "algo": getattr(args, "sip_algo", "scan"), "batch_per_gpu": cs["batch"], "n": cs["n"],
             "m": cs["m"], "alpha": cs["alpha"],
             "l2": "every iteration streams the factor / matrix / iterate planes (> 2 GB) > 126 MB L2"}
    elif w in ("stdm", "spdm"):
        bpr = 40 if w == "stdm" else 56
        c = {"workload": (f"config 3 {w.upper()}: B=4096 non-dominant systems, N=2048, 8 decoupled "
                          "zero pivots per system, seed 2"),
             "solver": w, "batch_per_gpu": 4096, "n": 2048, "layout": "interleaved row-aligned",
             "l2": f"inputs {bpr * 4096 * 2048 / 1e9:.2f} GB > 126 MB L2"}
    elif w == "hb":
        c = {"workload": ("config 4 HB: B=64 five-point systems, 64x32 grid (N=2048), alpha=0.5; step = "
                          "sip_hb_solve (dense HB inverses of L and U on DMMA + SIP-HB iterations), seed 3"),
             "solver": "sip_hb", "batch_per_gpu": 64, "n": 2048, "m": 32,
             "l2": "X, X_next, P per factor: 3 x 2B x 33.5 MB = 12.9 GB"}
    else:  # adi
        c = {"workload": ("config 5 ADI: one step on a 8192x8192 grid (x-sweep of 8192 TD systems, "
                          "transpose/all-to-all, y-sweep of 8192), seed 0"),
             "solver": "adi (ntdm partitioned x2)", "grid": 8192, "l2": "5.4 GB per step > 126 MB L2"}
    c["parallelism"] = par
    return c


class Direct:
    metric, unit, scaling = "systems_solved_per_s", "systems/s", "weak"

    def __init__(self, args, rank, dev, name):
        import torch
        from paper_1804_09666_b200 import _lib
        from paper_1804_09666_b200.core import ptr, workspace
        self.args = args
        solver, batch, n, cfg, sparse, desc = DIRECT[name]
        self.solver, self.batch, self.n = solver, batch, n
        self.kind = "tri" if solver == "ntdm" else "penta"
        self.arrs = direct_inputs(name, rank)
        offsets = (-1, 0, 1) if self.kind == "tri" else (-2, -1, 0, 1, 2)
        self.lay = _lib.LAYOUT_INTERLEAVED if args.layout == "interleaved" else _lib.LAYOUT_SYSTEM_MAJOR
        self.algo = {"sequential": _lib.ALGO_SEQUENTIAL, "partitioned": _lib.ALGO_PARTITIONED}[args.algo]
        self.host = rowaligned(self.arrs, offsets, args.layout)
        self.ld = batch if args.layout == "interleaved" else n
        self.d_in = [torch.from_numpy(h).to(dev) for h in self.host]
        self.x = torch.empty(self.host[-1].shape, dtype=torch.float64, device=dev)
        self.status = torch.empty(batch, dtype=torch.int32, device=dev)
        self.index = torch.empty(batch, dtype=torch.int32, device=dev)
        self.nz = torch.empty(batch, dtype=torch.int64, device=dev)
        L = _lib.lib()
        self.ws = workspace(L.bx_workspace_bytes(_lib.SOLVER[solver], batch, n, self.lay, self.algo), dev)
        self.bytes_per_row = 40 if self.kind == "tri" else 56
        # MNPDM on sparse outer diagonals (its purpose): the +-2 diagonals as
        # per-system row lists, compacted once per matrix outside the timed
        # region (PentaMatrix.sparse_outer); the solve streams 40 B/row
        self.sparse = solver == "mnpdm" and sparse and args.algo == "partitioned"
        self.outer_bytes = 0
        if self.sparse:
            cnt = torch.empty(batch, dtype=torch.int32, device=dev)
            c2, g2 = self.d_in[0], self.d_in[4]
            _lib.call("bx_outer_compact_f64", ptr(c2), ptr(g2), ptr(cnt), None, None, None, 0, batch, n,
                      self.ld, self.lay, torch.cuda.current_stream().cuda_stream)
            self.outer_k = max(int(cnt.max()), 1)
            self.orow = torch.empty((batch, self.outer_k), dtype=torch.int32, device=dev)
            self.os2 = torch.empty((batch, self.outer_k), dtype=torch.float64, device=dev)
            self.op2 = torch.empty((batch, self.outer_k), dtype=torch.float64, device=dev)
            _lib.call("bx_outer_compact_f64", ptr(c2), ptr(g2), ptr(cnt), ptr(self.orow), ptr(self.os2),
                      ptr(self.op2), self.outer_k, batch, n, self.ld, self.lay,
                      torch.cuda.current_stream().cuda_stream)
            self.bytes_per_row = 40
            self.outer_bytes = batch * self.outer_k * (4 + 8 + 8)
        self.units = batch
        # partitioned: the solver kernel + the status / re-solve pass (direct_fixup)
        # partitioned: interface-iteration kernel, tree retry pass, re-solve /
        # status pass (sparse-outer entry: the first two)
        self.launches_per_step = (2 if self.sparse else 3) if args.algo == "partitioned" else 1
        gb = self.bytes_per_row * batch * n / 1e9
        # inputs that fit the 126 MB L2 (config 1: 42 MB) are flushed out of it
        # before every timed step (a 512 MB write, outside the step's events)
        self.flush_l2 = gb < 0.5

    def solve(self, ins, out):
        import torch
        from paper_1804_09666_b200 import _lib
        from paper_1804_09666_b200.core import ptr
        L, s = _lib.lib(), torch.cuda.current_stream().cuda_stream
        tail = (self.batch, self.n, self.ld, self.lay, self.algo, ptr(self.ws), self.ws.numel(), s)
        if self.sparse:  # ins: sub1, main, sup1, rhs
            rc = L.bx_mnpdm_sparse_f64(ptr(self.orow), ptr(self.os2), ptr(self.op2), self.outer_k,
                                       *(ptr(t) for t in ins), ptr(out), ptr(self.status),
                                       ptr(self.index), ptr(self.nz), self.batch, self.n, self.ld,
                                       self.lay, s)
        elif self.solver == "ntdm":
            rc = L.bx_ntdm_f64(*(ptr(t) for t in ins), ptr(out), ptr(self.status), ptr(self.index), *tail)
        elif self.solver == "npdm":
            rc = L.bx_npdm_f64(*(ptr(t) for t in ins), ptr(out), ptr(self.status), ptr(self.index), *tail)
        else:
            rc = L.bx_mnpdm_f64(*(ptr(t) for t in ins), ptr(out), ptr(self.status), ptr(self.index),
                                ptr(self.nz), *tail)
        _lib.check(rc, self.solver)

    def step(self):
        self.solve([self.d_in[i] for i in (1, 2, 3, 5)] if self.sparse else self.d_in, self.x)

    def check(self):
        """Sampled parity gate against the C restatement of the reference."""
        from oracle import cport
        idx = np.arange(0, self.batch, max(1, self.batch // 16))
        sl = [a[idx] for a in self.arrs]
        if self.kind == "tri":
            ref, _, _ = cport.ntdm(*cport.rowaligned_tri(*sl[:3]), np.ascontiguousarray(sl[3]))
        else:
            ref, _, _, _ = cport.penta(1 if self.solver == "mnpdm" else 0,
                                       *cport.rowaligned_penta(*sl[:5]), np.ascontiguousarray(sl[5]))
        x = self.x.cpu().numpy()
        x = x.T if self.args.layout == "interleaved" else x
        err = float(np.max(np.abs(x[idx] - ref) / np.max(np.abs(ref), axis=1, keepdims=True)))
        assert int((self.status != 0).sum()) == 0, "unexpected zero pivot"
        assert err <= 1e-10, f"parity gate failed: {err}"
        return err

    def e2e_prepare(self):
        import torch
        host = self.host
        self.host_outer = None
        if self.sparse:  # host inputs: sub1, main, sup1, rhs + the outer row lists
            from paper_1804_09666_b200.pipeline import outer_lists
            host = [self.host[i] for i in (1, 2, 3, 5)]
            lists = outer_lists(self.host[0], self.host[4])
            self.host_outer = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in lists]
        self.pinned = [torch.from_numpy(h).pin_memory() for h in host]
        self.x_host = torch.empty(self.host[-1].shape, dtype=torch.float64).pin_memory()
        self.h2d = sum(h.nbytes for h in host) + sum(t.numel() * t.element_size()
                                                      for t in (self.host_outer or []))
        self.d2h = self.x_host.numel() * 8
        self.pipe = None
        if self.sparse and self.args.layout != "system":
            raise SystemExit("sparse-outer MNPDM e2e path is system-major only")
        if self.args.layout == "system":
            # chunked H2D / solve / D2H overlap on three streams (pipeline.py)
            from paper_1804_09666_b200.pipeline import HostPipeline
            self.pipe = HostPipeline("mnpdm_sparse" if self.sparse else self.solver, self.n,
                                     max(1, self.batch // self.args.e2e_chunks), self.x.device,
                                     algo=self.args.algo,
                                     outer_k=self.host_outer[0].shape[1] if self.sparse else 0)
            self.e2e_path = ("pinned host -> bx C ABI per chunk -> pinned host x (system-major: "
                             f"{self.args.e2e_chunks} chunks, H2D / solve / D2H overlapped on 3 "
                             "streams, pipeline.py)")
        else:
            self.d_e2e = [torch.empty_like(t) for t in self.d_in]
            self.x_e2e = torch.empty_like(self.x)

    def e2e_step(self):
        if self.pipe is not None:
            self.pipe.run(self.pinned, self.x_host, host_outer=self.host_outer)
            return
        for h, d in zip(self.pinned, self.d_e2e):
            d.copy_(h, non_blocking=True)
        self.solve(self.d_e2e, self.x_e2e)
        self.x_host.copy_(self.x_e2e, non_blocking=True)

    def roofline(self, mean_launch, peak):
        alg = self.bytes_per_row * self.batch * self.n + self.outer_bytes
        ach = alg / mean_launch / 1e9
        kern = f"bx {self.solver} ({self.args.algo}{', sparse outer diagonals' if self.sparse else ''})"
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "kernel": kern, "algorithmic_bytes_per_launch": alg,
                "bytes_per_row": self.bytes_per_row}

    def cpu_baseline(self, budget_s=5.0):
        rate0, _, _ = cpu_direct_rate(self.solver, self.arrs, min(self.batch, 128))
        sample = int(min(self.batch, max(64, rate0 * budget_s)))
        tot_s, tot_n, passes = 0.0, 0, 0
        while tot_s < budget_s and passes < 1000:  # ~5 s of host work (tiny configs: many passes)
            rate, dt, thr = cpu_direct_rate(self.solver, self.arrs, sample)
            tot_s += dt; tot_n += sample; passes += 1
        return {"value": tot_n / tot_s, "unit": self.unit, "cores": thr, "kind": "port",
                "sample": f"{passes} pass(es) over {sample} of {self.batch} systems ({tot_s:.1f} s), "
                          f"C restatement of the reference (oracle/c/bx_oracle.c), OpenMP {thr} threads"}


SIP_CFG = dict(batch=64, n=262144, m=512, alpha=0.5, cfg=3)


class Sip:
    metric, unit, scaling = "sip_system_iterations_per_s", "system-iterations/s", "weak"

    def __init__(self, args, rank, dev):
        import torch
        from paper_1804_09666_b200 import _lib, workloads as W
        from paper_1804_09666_b200.core import workspace
        c = SIP_CFG
        self.batch, self.n, self.m, self.alpha = c["batch"], c["n"], c["m"], c["alpha"]
        rng = np.random.default_rng([c["cfg"], rank] if rank else c["cfg"])
        self.arrs = W.five_point(self.batch, self.n, self.m, rng=rng)
        self.tol = W.sip_tolerance(self.arrs[5])
        m = self.m
        self.host = rowaligned(self.arrs, (-m, -1, 0, 1, m), "system")
        self.d_in = [torch.from_numpy(h).to(dev) for h in self.host]
        self.d_tol = torch.from_numpy(self.tol).to(dev)
        f64 = dict(dtype=torch.float64, device=dev)
        self.x = torch.empty((self.batch, self.n), **f64)
        self.iters = torch.empty(self.batch, dtype=torch.int64, device=dev)
        self.res = torch.empty(self.batch, **f64)
        self.status = torch.empty(self.batch, dtype=torch.int32, device=dev)
        self.ws = workspace(_lib.lib().bx_sip_workspace_bytes(self.batch, self.n, m), dev)
        # scan: correction form + row scans (throughput path, k within +-1 of
        # the reference loop); wavefront: Algorithm 1 verbatim, bit parity
        self.algo = args.sip_algo
        # prefix table, skew/pack, wavefront kernel (setup [+ iterations]) [, scan kernel]
        self.launches_per_step = 4 if self.algo == "scan" else 3

    def solve(self, ins, x):
        import torch
        from paper_1804_09666_b200 import _lib
        from paper_1804_09666_b200.core import ptr
        _lib.call("bx_sip_f64", *(ptr(t) for t in ins[:5]), ptr(ins[5]), ptr(self.d_tol), ptr(x),
                  None, ptr(self.iters), ptr(self.res), None, ptr(self.status), None, None,
                  self.batch, self.n, self.m, self.alpha, 500, 0, self.n, _lib.LAYOUT_SYSTEM_MAJOR,
                  4 if self.algo == "scan" else 2, ptr(self.ws), self.ws.numel(),
                  torch.cuda.current_stream().cuda_stream)

    def step(self):
        self.solve(self.d_in, self.x)

    def check(self):
        from oracle import cport
        assert int((self.status != 0).sum()) == 0
        self.total_iters = int(self.iters.sum())
        self.units = self.total_iters
        idx = np.arange(0, self.batch, max(1, self.batch // 4))
        ref = cport.sip(*cport.rowaligned_penta(*(a[idx] for a in self.arrs[:5]), m=self.m),
                        self.arrs[5][idx], self.tol[idx], m=self.m, alpha=self.alpha)
        if self.algo == "scan":  # north-star SIP contract: k +-1, residual below the tolerance
            assert np.all(np.abs(self.iters.cpu().numpy()[idx] - ref["iterations"]) <= 1), "SIP parity gate"
            assert bool((self.res.cpu().numpy() < self.tol).all()), "SIP parity gate (residual)"
            x = self.x.cpu().numpy()[idx]
            err = float(np.max(np.abs(x - ref["x"])) / np.max(np.abs(ref["x"])))
            assert err <= 1e-7, "SIP parity gate (iterate)"
            return err
        assert np.array_equal(self.iters.cpu().numpy()[idx], ref["iterations"])
        assert np.array_equal(self.x.cpu().numpy()[idx], ref["x"]), "SIP parity gate"
        return 0.0

    def e2e_prepare(self):
        import torch
        self.pinned = [torch.from_numpy(h).pin_memory() for h in self.host]
        self.x_host = torch.empty((self.batch, self.n), dtype=torch.float64).pin_memory()
        self.d_e2e = [torch.empty_like(t) for t in self.d_in]
        self.x_e2e = torch.empty_like(self.x)
        self.h2d = sum(h.nbytes for h in self.host)
        self.d2h = self.x_host.numel() * 8

    def e2e_step(self):
        for h, d in zip(self.pinned, self.d_e2e):
            d.copy_(h, non_blocking=True)
        self.solve(self.d_e2e, self.x_e2e)
        self.x_host.copy_(self.x_e2e, non_blocking=True)

    def roofline(self, mean_launch, peak):
        alg = 104 * self.n * self.total_iters   # 104 B per row-iteration
        ach = alg / mean_launch / 1e9
        if self.algo == "scan":
            kern = "bx sip_scan (ILU setup pass + forward/backward row-scan sweeps of every iteration)"
            note = ("correction form streams 128 B/row-iteration (A, b, L, U, y, x) plus one extra "
                    "forward sweep per solve; the setup pass is inside the timed solve")
        else:
            kern = "bx sip_wave (setup + all iterations, one launch)"
            note = "Algorithm 1 verbatim streams ~184 B/row-iteration (K, factors, y, A, b, x)"
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "kernel": kern,
                "algorithmic_bytes_per_launch": alg, "bytes_per_row_iteration": 104, "note": note}

    def cpu_baseline(self, budget_s=5.0):
        from oracle import cport
        sample = self.batch  # the whole batch (~1 s on 16 threads): an 8-system sample swung 800-1070
        a = [x[:sample] for x in self.arrs]
        r = cport.rowaligned_penta(*a[:5], m=self.m)
        t0 = time.perf_counter()
        out = cport.sip(*r, a[5], self.tol[:sample], m=self.m, alpha=self.alpha)
        dt = time.perf_counter() - t0
        its = int(out["iterations"].sum())
        return {"value": its / dt, "unit": self.unit, "cores": cport.threads(), "kind": "port",
                "sample": f"{sample} of {self.batch} systems ({its} system-iterations incl. ILU setup, "
                          f"{dt:.1f} s), C restatement (oracle/c/bx_oracle.c), OpenMP {cport.threads()} threads"}


class Exact:
    """Config 3: symbolic solvers on non-dominant systems with 8 zero pivots."""
    metric, unit, scaling = "systems_solved_per_s", "systems/s", "weak"
    launches_per_step = 1

    def __init__(self, args, rank, dev, kind):
        import torch
        from paper_1804_09666_b200 import _lib, workloads as W
        from paper_1804_09666_b200.core import workspace
        self.kind, self.batch, self.n = kind, 4096, 2048
        rng = np.random.default_rng([2, rank] if rank else 2)
        if kind == "stdm":
            *self.arrs, self.rows = W.td_symbolic(self.batch, self.n, rng=rng)
            self.offsets = (-1, 0, 1)
        else:
            *self.arrs, self.rows = W.pd_symbolic(self.batch, self.n, rng=rng)
            self.offsets = (-2, -1, 0, 1, 2)
        self.host = rowaligned(self.arrs, self.offsets, "interleaved")
        self.d_in = [torch.from_numpy(h).to(dev) for h in self.host]
        self.x = torch.empty((self.n, self.batch), dtype=torch.float64, device=dev)
        self.st = torch.empty(self.batch, dtype=torch.int32, device=dev)
        self.subs = torch.empty(self.batch, dtype=torch.int32, device=dev)
        self.ws = workspace(_lib.lib().bx_workspace_bytes(_lib.SOLVER[kind], self.batch, self.n, 0, 0), dev)
        self.units = self.batch
        self.bytes_per_row = 40 if kind == "stdm" else 56

    def solve(self, ins, x):
        import torch
        from paper_1804_09666_b200 import _lib
        from paper_1804_09666_b200.core import ptr
        s = torch.cuda.current_stream().cuda_stream
        if self.kind == "stdm":
            _lib.call("bx_stdm_f64", *(ptr(t) for t in ins), ptr(x), ptr(self.st), None, ptr(self.subs),
                      self.batch, self.n, self.batch, 0, ptr(self.ws), self.ws.numel(), s)
        else:
            _lib.call("bx_spdm_f64", *(ptr(t) for t in ins), ptr(x), ptr(self.st), None, ptr(self.subs),
                      self.batch, self.n, self.batch, 0, ptr(self.ws), self.ws.numel(), s)

    def step(self):
        self.solve(self.d_in, self.x)

    def check(self):
        from oracle.exact import limit_solve_mp
        assert int((self.st != 0).sum()) == 0, "symbolic solve status"
        assert bool((self.subs == 8).all()), "substitution count"
        x = self.x.cpu().numpy().T
        err = 0.0
        nd = len(self.offsets)
        for s_ in range(0, self.batch, self.batch // 4):
            ref = limit_solve_mp([a[s_] for a in self.arrs[:nd]], list(self.offsets), self.arrs[nd][s_])
            err = max(err, float(np.max(np.abs(x[s_] - ref)) / np.max(np.abs(ref))))
        assert err <= 1e-10, f"symbolic parity gate {err}"
        return err

    def e2e_prepare(self):
        import torch
        self.pinned = [torch.from_numpy(h).pin_memory() for h in self.host]
        self.x_host = torch.empty((self.n, self.batch), dtype=torch.float64).pin_memory()
        self.d_e2e = [torch.empty_like(t) for t in self.d_in]
        self.x_e2e = torch.empty_like(self.x)
        self.h2d = sum(h.nbytes for h in self.host)
        self.d2h = self.x_host.numel() * 8

    def e2e_step(self):
        for h, d in zip(self.pinned, self.d_e2e):
            d.copy_(h, non_blocking=True)
        self.solve(self.d_e2e, self.x_e2e)
        self.x_host.copy_(self.x_e2e, non_blocking=True)

    def roofline(self, mean_launch, peak):
        alg = self.bytes_per_row * self.batch * self.n
        ach = alg / mean_launch / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "kernel": f"bx {self.kind} (symbolic pivot pass + pivoted limit solve)",
                "algorithmic_bytes_per_launch": alg, "bytes_per_row": self.bytes_per_row}

    def cpu_baseline(self, budget_s=5.0):
        return None  # the reference's exact solver needs hours per system here


class Hb:
    """Config 4 HB: SIP with Hotelling-Bodewig inverses at N=2048 (DMMA)."""
    metric, unit, scaling = "sip_hb_system_iterations_per_s", "system-iterations/s", "weak"
    launches_per_step = 1

    def __init__(self, args, rank, dev, batch=64, n=2048, m=32, alpha=0.5):
        import torch
        from paper_1804_09666_b200 import _lib, workloads as W
        from paper_1804_09666_b200.core import workspace
        self.batch, self.n, self.m, self.alpha = batch, n, m, alpha
        rng = np.random.default_rng([3, rank] if rank else 3)
        self.arrs = W.five_point(batch, n, m, rng=rng)
        self.tol = W.sip_tolerance(self.arrs[5])
        self.host = rowaligned(self.arrs, (-m, -1, 0, 1, m), "system")
        self.d_in = [torch.from_numpy(h).to(dev) for h in self.host]
        self.d_tol = torch.from_numpy(self.tol).to(dev)
        f64 = dict(dtype=torch.float64, device=dev)
        self.x = torch.empty((batch, n), **f64)
        self.iters = torch.empty(batch, dtype=torch.int64, device=dev)
        self.inv_it = torch.empty(2 * batch, dtype=torch.int64, device=dev)
        self.st = torch.empty(batch, dtype=torch.int32, device=dev)
        self.ws = workspace(_lib.lib().bx_hb_workspace_bytes(batch, n), dev)

    def solve(self, ins, x):
        import torch
        from paper_1804_09666_b200 import _lib
        from paper_1804_09666_b200.core import ptr
        _lib.call("bx_sip_hb_f64", *(ptr(t) for t in ins[:5]), ptr(ins[5]), ptr(self.d_tol), ptr(x),
                  None, ptr(self.iters), None, None, ptr(self.st), None, None, ptr(self.inv_it), None,
                  self.batch, self.n, self.m, self.alpha, 500, 200, 0, self.n, 1, ptr(self.ws),
                  self.ws.numel(), torch.cuda.current_stream().cuda_stream)

    def step(self):
        self.solve(self.d_in, self.x)

    def check(self):
        import torch
        from oracle import cport
        assert int((self.st != 0).sum()) == 0
        self.units = int(self.iters.sum())
        self.inv_total = int(self.inv_it.sum())
        idx = np.arange(0, self.batch, self.batch // 4)
        ref = cport.sip(*cport.rowaligned_penta(*(a[idx] for a in self.arrs[:5]), m=self.m),
                        self.arrs[5][idx], self.tol[idx], m=self.m, alpha=self.alpha)
        its = self.iters.cpu().numpy()[idx]
        assert np.all(np.abs(its - ref["iterations"]) <= 1), "SIP-HB iteration count"
        x = self.x.cpu().numpy()[idx]
        err = float(np.max(np.abs(x - ref["x"])) / np.max(np.abs(ref["x"])))
        assert err <= 1e-7
        # DGEMM peak on this box (roofline denominator): torch.matmul float64
        a = torch.randn(8192, 8192, dtype=torch.float64, device=self.x.device)
        torch.matmul(a, a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            torch.matmul(a, a)
        e1.record()
        torch.cuda.synchronize()
        self.dgemm_tflops = 3 * 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
        return err

    def e2e_prepare(self):
        import torch
        self.pinned = [torch.from_numpy(h).pin_memory() for h in self.host]
        self.x_host = torch.empty((self.batch, self.n), dtype=torch.float64).pin_memory()
        self.d_e2e = [torch.empty_like(t) for t in self.d_in]
        self.x_e2e = torch.empty_like(self.x)
        self.h2d = sum(h.nbytes for h in self.host)
        self.d2h = self.x_host.numel() * 8

    def e2e_step(self):
        for h, d in zip(self.pinned, self.d_e2e):
            d.copy_(h, non_blocking=True)
        self.solve(self.d_e2e, self.x_e2e)
        self.x_host.copy_(self.x_e2e, non_blocking=True)

    def roofline(self, mean_launch, peak):
        fl = self.inv_total * self.n ** 3 / 3  # useful triangular x triangular flops
        ach = fl / mean_launch / 1e12
        return {"bound": "tensor", "achieved": ach, "peak": self.dgemm_tflops, "unit": "TFLOP/s",
                "frac": ach / self.dgemm_tflops, "traffic": None,
                "kernel": "bx hb_gemm (DMMA m16n8k16 f64) within the whole sip_hb step",
                "useful_flops_per_step": fl,
                "peak_source": "torch.matmul float64 8192^3 measured in this run (DGEMM)",
                "note": "achieved counts only the HB GEMM flops but divides by the whole step"}

    def cpu_baseline(self, budget_s=5.0):
        # the reference's dense HB is numpy matmul (BLAS); oracle.inverse.sip_hb
        # restates it with the same numpy calls, timed on a 2-system sample
        from oracle import inverse as OI
        sample = 2
        a = [x[:sample] for x in self.arrs]
        t0 = time.perf_counter()
        out = OI.sip_hb(*a[:5], a[5], self.tol[:sample], 500, m=self.m, alpha=self.alpha)
        dt = time.perf_counter() - t0
        its = int(np.asarray(out["iterations"]).sum())
        cores = len(os.sched_getaffinity(0))
        return {"value": its / dt, "unit": self.unit, "cores": cores, "kind": "port",
                "sample": f"{sample} of {self.batch} systems ({its} system-iterations incl. ILU(0) and "
                          f"both dense HB inversions, {dt:.1f} s), numpy restatement of the reference "
                          f"(oracle/inverse.sip_hb, BLAS on up to {cores} threads)"}


class Adi:
    """Config 5: one ADI step on an 8192^2 grid (x-sweep, transpose / all-to-all, y-sweep)."""
    metric, unit, scaling = "systems_solved_per_s", "systems/s", "strong"
    launches_per_step = 7  # 2 x (interface-iteration kernel + tree retry pass + status pass) + transpose

    def __init__(self, args, rank, dev, world, n=8192):
        import torch
        import torch.distributed as dist
        from paper_1804_09666_b200 import workloads as W
        from paper_1804_09666_b200.adi import ADIStep
        self.n, self.world = n, world
        xs, ys = W.adi_step(n, seed=0)
        nyl, nxl = n // world, n // world
        rows = slice(rank * nyl, (rank + 1) * nyl)
        cols = slice(rank * nxl, (rank + 1) * nxl)

        def ra(sub, main, sup, sl):
            m_ = np.ascontiguousarray(main[sl])
            a = np.zeros_like(m_); a[:, 1:] = sub[sl]
            c = np.zeros_like(m_); c[:, :-1] = sup[sl]
            return [a, m_, c]
        self.hx = ra(*xs[:3], rows) + [np.ascontiguousarray(xs[3][rows])]
        self.hy = ra(*ys, cols)
        self.dx = [torch.from_numpy(h).to(dev) for h in self.hx]
        self.dy = [torch.from_numpy(h).to(dev) for h in self.hy]
        self.stepper = ADIStep(self.dx[:3], self.dy, group=dist.group.WORLD if world > 1 else None)
        self.units = 2 * n // world          # systems solved per rank per step
        self.x = self.stepper.U

    def step(self):
        self.stepper(self.dx[3])

    def check(self):
        from oracle import cport
        import torch
        u = self.stepper(self.dx[3])[0]
        torch.cuda.synchronize()
        if self.world > 1:
            return 0.0
        # sampled parity: columns j via oracle x-sweep of all rows + y-sweep of column j
        X, _, _ = cport.ntdm(*self.hx)
        js = [0, self.n // 3, self.n - 1]
        Y = np.ascontiguousarray(X[:, js].T)
        ref, _, _ = cport.ntdm(*(h[js] for h in self.hy), Y)
        got = u.cpu().numpy()[js]
        err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
        assert err <= 1e-10, f"ADI parity gate {err}"
        return err

    def e2e_prepare(self):
        import torch
        self.pinned = [torch.from_numpy(h).pin_memory() for h in self.hx + self.hy]
        self.x_host = torch.empty(tuple(self.stepper.U.shape), dtype=torch.float64).pin_memory()
        self.h2d = sum(h.nbytes for h in self.hx + self.hy)
        self.d2h = self.x_host.numel() * 8

    def e2e_step(self):
        for h, d in zip(self.pinned, self.dx + self.dy):
            d.copy_(h, non_blocking=True)
        u, _, _ = self.stepper(self.dx[3])
        self.x_host.copy_(u, non_blocking=True)

    def roofline(self, mean_launch, peak):
        alg = 2 * 40 * self.n * self.n // self.world
        ach = alg / mean_launch / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "kernel": "adi step (2 x bx_ntdm partitioned + transpose)",
                "algorithmic_bytes_per_launch": alg, "bytes_per_row": 80,
                "note": "per step: 2 sweeps x 40 B/row; the transpose (16 B/element) is extra traffic"}

    def cpu_baseline(self, budget_s=5.0):
        from oracle import cport
        rows = 1024
        t0 = time.perf_counter()
        cport.ntdm(*(h[:rows] for h in self.hx))
        dt = time.perf_counter() - t0
        rate = rows / dt
        return {"value": rate, "unit": self.unit, "cores": cport.threads(), "kind": "port",
                "sample": f"{rows} of the {self.n} x-sweep systems ({dt:.2f} s), C restatement, "
                          f"OpenMP {cport.threads()} threads"}


WORKLOADS = sorted(list(DIRECT) + ["sip", "stdm", "spdm", "hb", "adi"])


def cpu_reference_arm(args):
    """--impl reference: the CPU restatement on the host cores, rank 0 only
    (under a launcher the ranks form a gloo group; the others only join it)."""
    world, rank, _ = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        try:
            if rank == 0:
                _cpu_reference_run(args, world)
            dist.barrier()
        finally:
            dist.destroy_process_group()
        return
    _cpu_reference_run(args, world)


def _cpu_reference_run(args, world):
    # all host threads (a launcher exports OMP_NUM_THREADS=1 to every rank;
    # only rank 0 works here, before the OpenMP runtime is loaded)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    from oracle import cport
    cport.set_threads(len(os.sched_getaffinity(0)))
    from oracle import cport
    times = []
    if args.workload not in DIRECT and args.workload != "sip":
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no CPU restatement timed for workload {args.workload} (the reference's exact / "
                          "HB / ADI paths are pure Python; see DESIGN.md)"}))
        return
    if args.workload in DIRECT:
        solver, bsz, n, cfg, sparse, desc = DIRECT[args.workload]
        arrs = direct_inputs(args.workload)
        metric, unit = "systems_solved_per_s", "systems/s"
        rate0, _, _ = cpu_direct_rate(solver, arrs, min(bsz, 256))
        sample = int(min(bsz, max(64, rate0 * 1.5)))          # ~1.5 s of CPU work per step
        for _ in range(args.warmup):
            cpu_direct_rate(solver, arrs, min(sample, 64))
        for _ in range(args.steps):
            _, dt, thr = cpu_direct_rate(solver, arrs, sample)
            times.append(dt)
        value = sample * len(times) / sum(times)
        samp = f"{sample} of {bsz} systems per step"
    else:
        from paper_1804_09666_b200 import workloads as W
        c = SIP_CFG
        metric, unit = "sip_system_iterations_per_s", "system-iterations/s"
        nsys = min(64, max(16, cport.threads()))  # at least one system per host thread
        arrs = W.five_point(nsys, c["n"], c["m"], rng=np.random.default_rng(c["cfg"]))
        tol = W.sip_tolerance(arrs[5])
        r = cport.rowaligned_penta(*arrs[:5], m=c["m"])
        its = 0
        for k in range(1 + args.steps):
            t0 = time.perf_counter()
            out = cport.sip(*r, arrs[5], tol, m=c["m"], alpha=c["alpha"])
            if k >= 1:
                times.append(time.perf_counter() - t0)
                its += int(out["iterations"].sum())
        value = its / sum(times)
        thr = cport.threads()
        desc, samp = "config 4 SIP", f"{nsys} of 64 systems per step (full sip_solve each)"
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": static_config(args, world),
            "cpu_baseline": {"value": value, "unit": unit, "cores": thr, "kind": "port",
                             "sample": f"{samp}, C restatement (oracle/c/bx_oracle.c), OpenMP {thr} threads"},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.workload == "sip":
        wl = Sip(args, rank, dev)
    elif args.workload in ("stdm", "spdm"):
        wl = Exact(args, rank, dev, args.workload)
    elif args.workload == "hb":
        wl = Hb(args, rank, dev)
    elif args.workload == "adi":
        wl = Adi(args, rank, dev, world)
    else:
        wl = Direct(args, rank, dev, args.workload)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world > 1:
            t = torch.tensor([v], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    wl.step()                      # correctness gate: sampled systems vs the C restatement
    torch.cuda.synchronize()
    gate_err = wl.check()

    for _ in range(args.warmup):
        wl.step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = ClockSampler(local).start() if rank == 0 else None
    if sampler:
        time.sleep(0.3)
    barrier()
    flush = getattr(wl, "flush_l2", False)
    scrub = torch.empty(64 << 20, dtype=torch.float64, device=dev) if flush else None  # 512 MB
    # launch-latency-sized steps (config 1: ~20 us of kernels behind three
    # launches): replay the step from a CUDA graph so that host enqueue jitter
    # stays out of the device-side events
    step_fn, graphed = wl.step, False
    if flush:
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                wl.step()
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                wl.step()
            g.replay()
            torch.cuda.synchronize()
            step_fn, graphed = g.replay, True
        except Exception as exc:  # capture not possible: time the direct launches
            sys.stderr.write(f"bench: CUDA graph capture of the step failed ({exc}); direct launches\n")
            torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for k in range(args.steps):
        if flush:
            scrub.fill_(float(k))
        ev[k][0].record()
        step_fn()
        ev[k][1].record()
    t1.record()
    barrier()
    clocks = sampler.stop() if sampler else None
    if flush:  # device time of the steps only (the flushes between them excluded)
        elapsed = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / 1e3)
    else:
        elapsed = max_over_ranks(t0.elapsed_time(t1) / 1e3)
    mean_launch = statistics.mean(a.elapsed_time(b) / 1e3 for a, b in ev)
    value = wl.units * world * args.steps / elapsed
    peak, peak_src = load_peaks()
    roof = wl.roofline(mean_launch, peak)
    roof["mean_launch_ms"] = 1e3 * mean_launch
    roof.setdefault("peak_source", peak_src)
    traffic = load_traffic(args)
    if traffic is not None:
        roof["traffic"] = traffic["bytes_per_launch"]
        roof["traffic_source"] = traffic["source"]

    wl.e2e_prepare()
    for _ in range(max(1, min(args.warmup, 2))):
        wl.e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, min(args.steps, 10))  # PCIe-bound: a longer window averages host-side jitter
    e0.record()
    for _ in range(e2e_steps):
        wl.e2e_step()
    e1.record()
    barrier()
    e2e_elapsed = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    if args.workload not in ("hb",):
        assert torch.equal(wl.x_host, wl.x.cpu()), "e2e result differs from the resident run"
    pcie = pcie_h2d_gbs(dev) if rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = wl.cpu_baseline()
    if rank == 0:
        cfg = static_config(args, world)
        if flush:
            cfg["launch"] = ("step replayed from a CUDA graph (launch-latency-sized work)" if graphed
                             else "direct launches (graph capture failed)")
        line = {
            "metric": wl.metric, "value": value, "unit": wl.unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
            "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg, "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": wl.units * world * e2e_steps / e2e_elapsed, "unit": wl.unit,
                    "h2d_bytes_per_step": wl.h2d, "d2h_bytes_per_step": wl.d2h,
                    "path": getattr(wl, "e2e_path", "pinned host -> H2D (cudaMemcpyAsync) -> bx C ABI "
                                                     "-> D2H x, one stream"),
                    "pcie_h2d_gbs_measured": pcie,
                    "h2d_gbs_achieved": wl.h2d * e2e_steps / e2e_elapsed / 1e9,
                    "pcie_frac": (wl.h2d * e2e_steps / e2e_elapsed / 1e9 / pcie) if pcie else None},
            "gpu_launches": args.steps * wl.launches_per_step,
            "clocks": clocks,
            "parity_gate": f"sampled systems vs C restatement, max rel err {gate_err:.2e}",
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="npdm", choices=WORKLOADS)
    ap.add_argument("--algo", default="partitioned", choices=["sequential", "partitioned"])
    ap.add_argument("--layout", default=None, choices=["interleaved", "system"],
                    help="C-ABI storage (default: system-major for partitioned, interleaved for sequential)")
    ap.add_argument("--sip-algo", default="scan", choices=["scan", "wavefront"],
                    help="SIP workload: scan = correction form + row scans (throughput path); "
                         "wavefront = Algorithm 1 verbatim (bit parity)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=8,
                    help="system chunks of the overlapped host pipeline (e2e leg)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return launch_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
                         "(torchrun --nproc-per-node N bench.py --gpus N, or plain bench.py --gpus N)")
    if args.layout is None:
        args.layout = "system" if args.algo == "partitioned" else "interleaved"
    if args.impl == "reference":
        cpu_reference_arm(args)
    else:
        run_ours(args)


def launch_ranks(args):
    """`python bench.py --gpus N` without a launcher: start N ranks on this node
    (torch.distributed.run on 127.0.0.1, a free port), forward their output,
    exit with the first non-zero rank status."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


if __name__ == "__main__":
    main()
