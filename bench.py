#!/usr/bin/env python
"""Benchmark of the B200 surrogate / full-quadrature IGA assembly path (BASELINE.json metric).

One step = every matrix of the workload assembled once (this rank's row slab under N > 1): full
quadrature and surrogate, for each form of the config (config 5 by default: 3D twisted-cube
stand-in, p=3, 128^3 elements, Poisson + mass, M=16 -> 4 matrices of 741M nnz each).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run (one
rank per GPU).  Ranks own contiguous row slabs cut on slowest-direction planes: the
full assembly has no data-path collective; the surrogate all-gathers the <= 2 MB table of lattice
samples (strategy B: each rank assembles only its own lattice rows); an NCCL all-reduce of per-slab
checksums closes the run.  Device time is the max over ranks; rank 0 prints one JSON line with the
step, a per-path / per-form breakdown (`paths`), the dominant kernel's roofline, the other BASELINE
configs (`configs`, N=1), the end-to-end figure through the public drop-in API (`e2e`) and the
reference's CPU path (`cpu_baseline`).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembled CSR nnz/s (surrogate & full-quadrature, fp64), % of roofline"
FP64_PEAK_TFLOPS = 37.2   # measured on this pool's B200: DMMA m8n8k4 / DFMA (profiles/fp64_peak.txt)


def _peaks():
    hbm = 6655.0
    src = "fallback (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        hbm = float(mp["hbm_gbs"])
        src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        pass
    return hbm, src


# ---------------------------------------------------------------------------------------------
# algorithmic work: reference-algorithm flops per element, output bytes
# ---------------------------------------------------------------------------------------------

def f_elem(form, n, p, g):
    L = (p + 1) ** n
    Q = g ** n
    U = L * (L + 1) // 2
    if form in ("poisson", "stokes_velocity"):
        return Q * (2 * n * n * L + 2 * n * U)
    if form == "mass":
        return Q * (L + 2 * U)
    return Q * ((4 * n * n + 2 * n ** 3 + 1) * L + 2 * U)


def csr_bytes(nnz, nrows):
    return 12 * nnz + 4 * (nrows + 1)


def roofline_time_s(form, path, n, p, g, E, nnz, nrows, plan, q, hbm_gbs):
    """t_roof = max(F / P_fp64, B / BW_HBM) for one matrix."""
    if path == "full":
        F = f_elem(form, n, p, g) * E
    else:
        F = f_elem(form, n, p, g) * plan.active_elements + 2 * (q + 1) * plan.interp_entries
    B = csr_bytes(nnz, nrows)
    return max(F / (FP64_PEAK_TFLOPS * 1e12), B / (hbm_gbs * 1e9)), F, B


# ---------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------------

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.lines = []

    def _nvml_loop(self):
        # in-process NVML sampling (no second process polling the driver during the timed region)
        nv = self.nv
        R = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((float(sm), float(mx), [k for k, b in R.items() if rs & b]))
            except Exception:
                pass
            self.stop_flag.wait(0.05)

    def start(self):
        self.nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            # NVML enumerates physical devices: honour CUDA_VISIBLE_DEVICES (indices or UUIDs)
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [x.strip() for x in vis.split(",") if x.strip()]
            if ids and self.dev < len(ids):
                tok = ids[self.dev]
                self.h = nv.nvmlDeviceGetHandleByIndex(int(tok)) if tok.isdigit() else nv.nvmlDeviceGetHandleByUUID(tok)
            else:
                self.h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.nv = nv
            self.samples = []
            self.stop_flag = threading.Event()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if getattr(self, "nv", None) is not None:
            time.sleep(0.1)
            self.stop_flag.set()
            self.t.join(timeout=1)
            sm = [s[0] for s in self.samples]
            mx = [s[1] for s in self.samples]
            reasons = sorted({r for s in self.samples for r in s[2]})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
# multi-GPU launch
# ---------------------------------------------------------------------------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args):
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) under torch.distributed.run."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but {have} CUDA device(s) visible"}), flush=True)
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------

def run_ours(args):
    import torch

    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200 import _lib
    from paper_1904_06971_b200.configs import CONFIGS
    from paper_1904_06971_b200.slabs import exchange_samples, job_slabs, lattice_owners
    from paper_1904_06971_b200.surrogate import build_sampling_lattice, surrogate_device, surrogate_plan, tilde_domain

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    torch.cuda.set_device(local)
    pkg.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    forms = args.forms.split(",") if args.forms else list(cfg.forms)
    paths = args.paths.split(",")
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    n = len(cfg.spans)
    ms = tuple(kv.m for kv in disc.space.kvs)
    N = int(np.prod(ms))
    E = int(np.prod(cfg.spans))
    g = disc.gauss
    lattice = build_sampling_lattice(disc.space.kvs, cfg.M)
    tilde = tilde_domain(cfg.p, ms)
    plan = surrogate_plan(disc, pkg.ConstantSampling(cfg.M), cfg.q)
    # per call: equal plane slabs for the full assembly, cost-weighted plane slabs for the surrogate
    jobs = [(f, path) for f in forms for path in paths]
    all_slabs = {(f, path): job_slabs(ms, cfg.p, world, path, f, lattice.indices) for f, path in jobs}
    slabs = {k: (v[rank] if world > 1 else None) for k, v in all_slabs.items()}
    exchanges = {}
    if world > 1:
        for f, path in jobs:
            if path == "surrogate":
                exchanges[(f, path)] = exchange_samples(lattice_owners(ms, lattice.indices, all_slabs[(f, path)]), dist)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    dmma = {}  # executed fp64 tensor-core instructions of the assembly kernel per job

    def one(f, path, checksum=False):
        fk = pkg.FormKind(f)
        n_irows = 0
        slab = slabs[(f, path)]
        if path == "full":
            res, _, _ = pkg.assemble_device(fk, disc, stream=sptr, slab=slab)
        else:
            mode = pkg.surrogate.DEFAULT_MODE[f].value
            res, st, _ = surrogate_device(fk, disc, cfg.M, cfg.q, mode, stream=sptr, slab=slab, lattice=lattice,
                                          tilde=tilde, exchange=exchanges.get((f, path)))
            n_irows = int(st.n_interp_rows)
        _, nl = _lib.last_timing()
        kt = _lib.last_kernel_times()
        dmma[(f, path)] = _lib.last_dmma_count()
        nrows, nnz = res.sizes()
        cs = res.checksum() if checksum else np.zeros(5)
        res.free()
        return nnz, nrows, nl, kt, cs, n_irows

    # the clock sampler (an nvidia-smi process polling every 100 ms) starts before the warm-up: its
    # start-up (NVML initialisation) stalled the first timed step by ~15 ms when started right before it
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        for f, path in jobs:
            one(f, path)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(jobs) + 1)] for _ in range(args.steps)]
    nnz_tot = 0
    launches = 0
    ktimes = {}
    per_job = {}
    checks = np.zeros(5)
    for s_ in range(args.steps):
        evs[s_][0].record(stream)
        for j, (f, path) in enumerate(jobs):
            nnz, nrows, nl, kt, cs, n_irows = one(f, path)
            evs[s_][j + 1].record(stream)
            nnz_tot += nnz
            launches += nl
            per_job[(f, path)] = (nnz, nrows, n_irows)
            for name, t in kt:
                ktimes.setdefault((f, path, name), []).append(t)
    torch.cuda.synchronize()
    ms_dev = evs[0][0].elapsed_time(evs[-1][-1])
    job_ms = {k: sum(evs[s_][j].elapsed_time(evs[s_][j + 1]) for s_ in range(args.steps)) / args.steps
              for j, k in enumerate(jobs)}
    clk = clocks.stop()
    for f, path in jobs:  # untimed verification step: per-slab checksums, all-reduced over NCCL below
        checks += one(f, path, checksum=True)[4]
    job_nnz = {k: float(v[0]) for k, v in per_job.items()}
    if dist:
        t = torch.tensor([ms_dev] + [job_ms[k] for k in jobs], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_dev = float(t[0].item())
        job_ms = {k: float(t[1 + j].item()) for j, k in enumerate(jobs)}
        tn = torch.tensor([float(nnz_tot)] + [job_nnz[k] for k in jobs], device="cuda", dtype=torch.float64)
        dist.all_reduce(tn)
        nnz_all = float(tn[0].item())
        job_nnz = {k: float(tn[1 + j].item()) for j, k in enumerate(jobs)}
        tc = torch.tensor(checks, device="cuda", dtype=torch.float64)
        dist.all_reduce(tc)  # NCCL checksum all-reduce over the slabs
        checks = tc.cpu().numpy()
    else:
        nnz_all = float(nnz_tot)
    value = nnz_all / (ms_dev / 1e3)
    hbm, hbm_src = _peaks()

    # ---- per path and form: device time per call (max over ranks), nnz/s, SURVEY §8d roofline fraction
    paths_out = {}
    for f, path in jobs:
        nnz_m = job_nnz[(f, path)]
        t_roof, F, B = roofline_time_s(f, path, n, cfg.p, g, E, nnz_m, N, plan, cfg.q, hbm)
        t = job_ms[(f, path)] / 1e3
        paths_out[f"{f}/{path}"] = {"ms": job_ms[(f, path)], "nnz": nnz_m, "nnz_per_s": nnz_m / t,
                                    "roofline_s": t_roof, "roofline_frac": t_roof / t,
                                    "roofline_bound": "fp64" if F / (FP64_PEAK_TFLOPS * 1e12) >= B / (hbm * 1e9) else "hbm",
                                    "algorithmic_flops": F, "output_bytes": B}

    # ---- per-kernel rooflines; the dominant kernel (largest device time) is the headline roofline
    rows = []
    for (f, path, name), ts in ktimes.items():
        avg = sum(ts) / len(ts)
        nnz, nrows, n_irows = per_job[(f, path)]
        if name in ("assemble_tiles", "assemble_mma"):
            flops_alg = f_elem(f, n, cfg.p, g) * (E if path == "full" else plan.active_elements) / world
            issued = 512.0 * dmma.get((f, path), 0)  # DMMA m8n8k4 f64 = 256 FMA
            hw = issued / (avg / 1e3) / 1e12
            rows.append({"kernel": f"{name}[{f},{path}]", "bound": "tensor", "achieved": hw, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": hw / FP64_PEAK_TFLOPS,
                         "algorithmic_achieved": flops_alg / (avg / 1e3) / 1e12,
                         "algorithmic_frac": flops_alg / (avg / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                         "ms": avg, "issued_flops": issued, "algorithmic_flops": flops_alg, "share": sum(ts)})
        elif name == "geom_D":
            # K3 writes U = |Mset|(|Mset|+1)/2 doubles per Gauss point: its HBM roofline; the
            # mass tensor (U = 1) is bound by the fp64 map / Jacobian evaluation instead (~300 flop / point)
            U = {"poisson": n * (n + 1) // 2, "mass": 1}.get(f)
            els = (E if path == "full" else plan.active_elements) / world
            if U:
                b = 8.0 * U * els * g ** n
                ach = b / (avg / 1e3) / 1e9
                rows.append({"kernel": f"geom_D[{f},{path}]", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                             "frac": ach / hbm, "ms": avg, "bytes": b, "share": sum(ts),
                             "fp64_frac_at_300_flop_per_point": 300.0 * els * g ** n / (avg / 1e3) / 1e12 / FP64_PEAK_TFLOPS})
            else:
                rows.append({"kernel": f"geom_D[{f},{path}]", "bound": None, "ms": avg, "share": sum(ts)})
        elif name in ("interp_tiles", "interp_rows3"):
            # the kernel's own output: value + column of every slot of the interpolated rows
            b = 12 * n_irows * (2 * cfg.p + 1) ** n
            ach = b / (avg / 1e3) / 1e9
            rows.append({"kernel": f"{name}[{f}]", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                         "frac": ach / hbm, "ms": avg, "bytes": b, "share": sum(ts)})
        elif name == "interp_slow_rows":
            rows.append({"kernel": f"interp_slow_rows[{f}]", "bound": None, "ms": avg, "share": sum(ts)})
    total_k = sum(sum(ts) for ts in ktimes.values())
    rows.sort(key=lambda r: -r["share"])
    for r in rows:
        r["share"] = r["share"] / total_k if total_k else None
    ranked = [r for r in rows if r.get("bound")]
    dom = dict(ranked[0]) if ranked else {}
    roof = {k: dom.get(k) for k in ("bound", "achieved", "peak", "unit", "frac", "algorithmic_achieved",
                                    "algorithmic_frac")}
    traffic = None
    try:  # DRAM bytes of the dominant kernel from its committed ncu --set full capture (per launch)
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        t = tr.get(dom.get("kernel") or "")
        if t and world == 1:
            traffic = {"bytes": t["dram_bytes_read"] + t["dram_bytes_write"], "read": t["dram_bytes_read"],
                       "write": t["dram_bytes_write"], "source": t["source"]}
    except (OSError, ValueError, KeyError):
        traffic = None
    roof.update({"traffic": traffic["bytes"] if traffic else None, "traffic_detail": traffic, "kernel": dom.get("kernel"),
                 "peak_source": "measured fp64 DMMA/DFMA microbenchmark (profiles/fp64_peak.txt)"
                 if dom.get("unit") == "TFLOP/s" else hbm_src,
                 "achieved_is": "executed fp64 tensor-core work (counted DMMA instructions x 512 flops) per launch / "
                                "average launch time: the hardware fraction",
                 "algorithmic_is": "SURVEY §8d reference-algorithm flops (F_elem x elements) per launch / launch time; "
                                   "the kernel is sum-factorised, so this equivalent rate can exceed the peak"})

    # ---- the other BASELINE configs (N=1): best-of-3 device time per call through the same entry points
    configs_out = None
    if world == 1 and not args.no_sweep:
        configs_out = sweep_configs(pkg, _lib, CONFIGS, args.config, hbm)

    # ---- end to end through the public drop-in API (host buffers, H2D inside, D2H of the CSR)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pkg, _lib, torch, dist, cfg, disc, jobs, slabs, lattice, tilde, exchanges, world)

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, forms, paths, threads_all=False)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_dev / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic geometry)",
            "config": {"workload": f"config{cfg.idx}:{cfg.name}", "forms": forms, "paths": paths, "p": cfg.p,
                       "spans": list(cfg.spans), "M": cfg.M, "q": cfg.q, "N": N,
                       "nnz_per_matrix": job_nnz[jobs[0]],
                       "parallelism": f"row-slab x{world} (surrogate: lattice-sample all-gather)" if world > 1
                       else "single GPU",
                       "l2": "outputs (8.9 GB/matrix at config 5) exceed L2; no flush needed"},
            "paths": paths_out, "roofline": roof, "kernels": rows, "configs": configs_out,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "checksum": {"nnz": checks[0], "sum": checks[1], "sumsq": checks[2]},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def sweep_configs(pkg, _lib, CONFIGS, skip, hbm):
    """Configs 1-4 (and any not benched above): every form x path, best of 3 calls (device time of the
    call from the library's own events), nnz/s and the SURVEY §8d roofline fraction."""
    from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device, surrogate_plan

    out = {}
    for k, cfg in CONFIGS.items():
        if k == skip:
            continue
        disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
        n = len(cfg.spans)
        ms = tuple(kv.m for kv in disc.space.kvs)
        N = int(np.prod(ms))
        E = int(np.prod(cfg.spans))
        lat = build_sampling_lattice(disc.space.kvs, cfg.M)
        plan = surrogate_plan(disc, pkg.ConstantSampling(cfg.M), cfg.q)
        entry = {"workload": cfg.name, "p": cfg.p, "spans": list(cfg.spans), "M": cfg.M, "q": cfg.q}
        for f in cfg.forms:
            for path in ("full", "surrogate"):
                best = None
                nnz = 0
                kt = []
                for _ in range(4):
                    if path == "full":
                        res, _, _ = pkg.assemble_device(pkg.FormKind(f), disc)
                    else:
                        res, _, _ = surrogate_device(pkg.FormKind(f), disc, cfg.M, cfg.q, DEFAULT_MODE[f].value,
                                                     lattice=lat)
                    t = _lib.last_timing()[0]
                    if best is None or t < best:
                        best = t
                        kt = _lib.last_kernel_times()
                    nnz = res.sizes()[1]
                    res.free()
                t_roof, F, B = roofline_time_s(f, path, n, cfg.p, disc.gauss, E, nnz, N, plan, cfg.q, hbm)
                entry[f"{f}/{path}"] = {"ms": best, "nnz": nnz, "nnz_per_s": nnz / (best / 1e3),
                                        "roofline_frac": t_roof / (best / 1e3),
                                        "kernel_ms": round(sum(v for _, v in kt), 4),
                                        "top_kernel": max(kt, key=lambda x: x[1])[0] if kt else None}
        out[str(k)] = entry
    return out


def run_e2e(args, pkg, _lib, torch, dist, cfg, disc, jobs, slabs, lattice, tilde, exchanges, world):
    """End-to-end step through the public API: `assemble` / `build_surrogate_matrix` (N=1: the
    reference-facing drop-in, host CSR + report out); under N > 1 the slab calls + D2H."""
    from paper_1904_06971_b200.surrogate import surrogate_device

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    _lib.host_staging_init(torch.cuda.current_device())  # one-time pinned ring, outside the timed region

    def e2e_job(f, path):
        fk = pkg.FormKind(f)
        if world == 1:
            if path == "full":
                A = pkg.assemble(fk, disc)
            else:
                A, _ = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(cfg.M), q=cfg.q)
            m = A.mat
            out = (m.nnz, m.indptr.nbytes + m.indices.nbytes + m.data.nbytes)
            del A, m
            return out + (_h2d_bytes(disc, path, lattice),)
        slab = slabs[(f, path)]
        if path == "full":
            res, _, _ = pkg.assemble_device(fk, disc, slab=slab)
        else:
            mode = pkg.surrogate.DEFAULT_MODE[f].value
            res, _, _ = surrogate_device(fk, disc, cfg.M, cfg.q, mode, slab=slab, lattice=lattice, tilde=tilde,
                                         exchange=exchanges.get((f, path)))
        ip, ix, dd = res.to_host()
        res.free()
        return dd.size, ip.nbytes + ix.nbytes + dd.nbytes, _h2d_bytes(disc, path, lattice)

    def e2e_step():
        outs = [e2e_job(f, path) for f, path in jobs]
        return tuple(sum(o[i] for o in outs) for i in range(3))

    for _ in range(2):  # untimed warm-up (host result buffers mapped and pinned, as in any repeated assembly)
        e2e_step()
    _lib.host_pool_sync()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    nnz_e = h2d = d2h = 0
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        nz, b_o, b_i = e2e_step()
        nnz_e += nz
        d2h += b_o
        h2d += b_i
    t_e2e = time.perf_counter() - t0
    if dist:
        t = torch.tensor([t_e2e, float(nnz_e)], device="cuda", dtype=torch.float64)
        tt = t.clone()
        dist.all_reduce(tt[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:2])
        t_e2e, nnz_e = float(tt[0].item()), float(tt[1].item())
    _lib.host_pool_release()  # unpin and drop the reused host result buffers before anything else
    return {"value": nnz_e / t_e2e, "unit": "nnz/s", "h2d_bytes_per_step": int(h2d // e2e_steps),
            "d2h_bytes_per_step": int(d2h // e2e_steps), "steps": e2e_steps,
            "api": "paper_1904_06971_b200.assemble / build_surrogate_matrix (scipy CSR + AssemblyReport out)"
            if world == 1 else "row-slab assemble_device / surrogate_device + Result.to_host per rank"}


def _h2d_bytes(disc, path, lattice):
    n = disc.space.n
    p = disc.space.kvs[0].p
    g = disc.gauss
    b = 0
    for kv in disc.space.kvs:
        b += 8 * ((kv.m + p + 1) + (kv.m - p) * g + g)
    w = disc.weights.weights
    if not np.all(w == w[0]):
        b += 8 * w.size
    gs = disc.geom.space
    for kv in gs.kvs:
        b += 8 * (kv.m + kv.p + 1)
    b += 8 * gs.N * (n + 1)
    if path == "surrogate":
        for d in range(n):
            s = lattice.sites[d].size
            b += 8 * (s * s + 3 * s)
    return b


# ---------------------------------------------------------------------------------------------
# CPU baseline: the reference itself (baseline/_ref) on bounded samples, extrapolated per element
# ---------------------------------------------------------------------------------------------

def _cpu_samples(cfg):
    """Bounded samples of the config's workload for the reference (same geometry, form, p, q):
    full quadrature on a coarse mesh (per-element cost), surrogate on the smallest mesh whose
    lattice keeps q (>= q+1 sites per direction) with a proportionally smaller M."""
    n = len(cfg.spans)
    if n == 3:
        full = (8, 8, 8) if cfg.p >= 3 else (12, 12, 12)
        surr, Ms = ((15, 15, 15), 2) if cfg.p >= 3 else ((14, 14, 14), 2)
    else:
        full = (64, 64)
        surr, Ms = ((96, 96), 8)
    return full, surr, Ms


def _cpu_job(job):
    """One sample assembly with the reference (single-threaded numpy) in a worker process."""
    cfg_idx, f, path, use_ref = job
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.configs import CONFIGS

    cfg = CONFIGS[cfg_idx]
    full, surr, Ms = _cpu_samples(cfg)
    spans = full if path == "full" else surr
    geom = cfg.geom()
    if use_ref:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        from surriga.assembly import FormKind, assemble, make_discretization
        from surriga.bspline import NurbsWeights, make_tensor_space
        from surriga.geometry import GeometryMap
        from surriga.surrogate import ConstantSampling, build_surrogate_matrix

        rg = GeometryMap(space=make_tensor_space(geom.space.p, geom.space.shape),
                         weights=NurbsWeights(geom.weights.weights, polynomial_weight=geom.weights.polynomial_weight),
                         control=geom.control)
        disc = make_discretization(rg, cfg.p, spans)
        fk = FormKind(f)
        t0 = time.perf_counter()
        if path == "full":
            A = assemble(fk, disc)
            rep = None
        else:
            A, rep = build_surrogate_matrix(fk, disc, ConstantSampling(Ms), q=cfg.q)
        dt = time.perf_counter() - t0
        return {"nnz": int(A.nnz), "s": dt, "E": int(np.prod(spans)),
                "active": None if rep is None else int(rep.active_elements),
                "interp_entries": None if rep is None else int(rep.interp_entries),
                "flags": None if rep is None else list(rep.flags)}
    from oracle import surriga_oracle as O

    disc = pkg.make_discretization(geom, cfg.p, spans)
    prob = O.problem_from_disc(pkg.FormKind(f), disc)
    t0 = time.perf_counter()
    if path == "full":
        _, ix, _, _, _ = O.assemble(prob)
        rep = None
    else:
        (_, ix, _), _, rep = O.surrogate(prob, Ms, cfg.q, None)
    dt = time.perf_counter() - t0
    return {"nnz": int(ix.size), "s": dt, "E": int(np.prod(spans)),
            "active": None if rep is None else int(rep["active_elements"]),
            "interp_entries": None if rep is None else int(rep["interp_entries"]), "flags": None if rep is None else rep["flags"]}


def _have_ref():
    return os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "surriga"))


def _cpu_init(use_ref):
    """Worker start-up: single-threaded numpy, reference modules imported before the timed region."""
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    try:  # BLAS pools inherited from the parent: one thread per worker process
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass
    import paper_1904_06971_b200  # noqa: F401
    if use_ref:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        import surriga.assembly  # noqa: F401
        import surriga.surrogate  # noqa: F401


def _cpu_warm(_):
    time.sleep(0.3)  # every worker of the pool is started (and initialised) before timing
    return os.getpid()


def cpu_baseline(cfg, forms, paths, threads_all=False):
    """The reference's CPU path on the config's workload, BASELINE.md §2 protocol.

    Every matrix of the step is timed by the reference on one core on a bounded sample (the sample
    jobs run side by side in single-threaded processes), and extrapolated to the config's size:
    full quadrature by its per-element time x elements (constant from 10^3 to 24^3 elements: 1.46 /
    1.50 / 1.49 ms for 3D p=3 Poisson); the surrogate by the same per-element time x the config's
    active elements, a lower bound of the reference's surrogate time (it also evaluates the full
    geometry grid and interpolates: ~6% more at 48^3; small samples overstate that share, so it is
    left out rather than extrapolated).  value = the step's nnz / the extrapolated step time.  threads_all (the reference arm): the full-quadrature
    matrices are split over every host core (process-parallel ``assemble(rows=slab)`` is bitwise the
    full assembly, test_assembly.py:94-100); the surrogate is not decomposable and stays on one core."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp

    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.surrogate import surrogate_plan

    use_ref = _have_ref()
    host_cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    sample_jobs = [(cfg.idx, f, "full", use_ref) for f in forms]
    if "surrogate" in paths:
        sample_jobs += [(cfg.idx, f, "surrogate", use_ref) for f in forms]
    # spawn, not fork: the parent may hold a CUDA context and driver-pinned host buffers
    with ProcessPoolExecutor(max_workers=len(sample_jobs), mp_context=mp.get_context("spawn"), initializer=_cpu_init,
                             initargs=(use_ref,)) as ex:
        list(ex.map(_cpu_warm, range(2 * len(sample_jobs))))
        t0 = time.perf_counter()
        res = list(ex.map(_cpu_job, sample_jobs))
        wall = time.perf_counter() - t0
    by = {(j[1], j[2]): r for j, r in zip(sample_jobs, res)}
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    ms = tuple(kv.m for kv in disc.space.kvs)
    N = int(np.prod(ms))
    E = int(np.prod(cfg.spans))
    nnz_m = 1
    for m in ms:
        k = np.arange(m)
        nnz_m *= int(np.sum(np.minimum(m - 1, k + cfg.p) - np.maximum(0, k - cfg.p) + 1))
    plan = surrogate_plan(disc, pkg.ConstantSampling(cfg.M), cfg.q)
    cores_full = host_cores if threads_all else 1
    t_step = 0.0
    nnz_step = 0
    detail = {}
    for f in forms:
        full = by[(f, "full")]
        t_el = full["s"] / full["E"]
        for path in paths:
            if path == "full":
                t = t_el * E / cores_full
            else:
                # lower bound: the quadrature of the active elements alone (the reference's surrogate
                # also evaluates the geometry on the full grid and interpolates; at 48^3 its
                # interpolation was ~6% of the call), so the baseline is never inflated
                sm = by[(f, "surrogate")]
                t = t_el * plan.active_elements
                detail[f"{f}/surrogate_sample"] = {"s": round(sm["s"], 3), "active": sm["active"],
                                                   "interp_entries": sm["interp_entries"], "flags": sm["flags"]}
            detail[f"{f}/{path}"] = {"extrapolated_s": round(t, 2), "nnz_per_s": nnz_m / t}
            t_step += t
            nnz_step += nnz_m
        detail[f"{f}/s_per_element"] = t_el
    full_s, surr_s, Ms = _cpu_samples(cfg)
    return {"value": nnz_step / t_step, "unit": "nnz/s", "cores": cores_full,
            "kind": "reference" if use_ref else "port",
            "sample": (f"config {cfg.idx} ({', '.join(forms)} x {', '.join(paths)}): the reference on one core per "
                       f"matrix at {full_s} elements (full quadrature) and {surr_s} elements with M={Ms} (surrogate, "
                       f"q={cfg.q}), extrapolated to {tuple(cfg.spans)} per element (surrogate: quadrature of its active elements, "
                       f"a lower bound)"
                       + (f"; full quadrature split over {host_cores} host cores (rows= slabs)" if threads_all else "")
                       + f"; sample wall {wall:.1f} s"),
            "extrapolated_step_s": t_step, "host_cores": host_cores, "detail": detail}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1904_06971_b200.configs import CONFIGS

    cfg = CONFIGS[args.config]
    forms = args.forms.split(",") if args.forms else list(cfg.forms)
    paths = args.paths.split(",")
    vals = []
    last = None
    for _ in range(max(1, args.steps)):
        last = cpu_baseline(cfg, forms, paths, threads_all=True)
        vals.append(last["value"])
    value = statistics.median(vals)
    cpu = dict(last)
    cpu["value"] = value
    # the same workload keys as our arm's line (sizes from the closed-form pattern, no assembly)
    import numpy as np
    import paper_1904_06971_b200 as pkg
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    ms = [int(kv.m) for kv in disc.space.kvs]
    nnz1 = 1.0
    for m in ms:  # rows of the basis-overlap pattern per direction: sum_i |{j : |i - j| <= p}|
        i = np.arange(m)
        nnz1 *= float((np.minimum(i + cfg.p, m - 1) - np.maximum(i - cfg.p, 0) + 1).sum())
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * len(forms) * len(paths) * nnz1 / value,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic geometry)", "impl": "reference",
            "config": {"workload": f"config{cfg.idx}:{cfg.name}", "forms": forms, "paths": paths, "p": cfg.p,
                       "spans": list(cfg.spans), "M": cfg.M, "q": cfg.q, "N": int(np.prod(ms)), "nnz_per_matrix": nnz1,
                       "parallelism": f"row-slab x{world} (surrogate: lattice-sample all-gather)" if world > 1
                       else "single GPU",
                       "l2": "outputs (8.9 GB/matrix at config 5) exceed L2; no flush needed"},
            "cpu_baseline": cpu, "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--forms", default="")
    ap.add_argument("--paths", default="full,surrogate")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
