#!/usr/bin/env python
"""Benchmark of the B200 surrogate / full-quadrature IGA assembly path (BASELINE.json metric).

One step = every matrix of the workload assembled once on this rank's row slab: full quadrature
and surrogate, for each form of the config (config 5 by default: 3D twisted-cube stand-in,
p=3, 128^3 elements, Poisson + mass, M=16 -> 4 matrices of 741M nnz each).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

N > 1 runs under torchrun: one rank per GPU, contiguous row slabs cut on slowest-direction
planes, no data-path collective; an NCCL all-reduce of per-slab checksums closes every step and
the device time is the max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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
    src = "fallback"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        hbm = float(mp["hbm_gbs"])
        src = "measured"
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

    def start(self):
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
# our arm
# ---------------------------------------------------------------------------------------------

def run_ours(args):
    import torch

    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200 import _lib
    from paper_1904_06971_b200.configs import CONFIGS
    from paper_1904_06971_b200.surrogate import build_sampling_lattice, surrogate_device, surrogate_plan, tilde_domain

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pkg.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    cfg = CONFIGS[args.config]
    forms = args.forms.split(",") if args.forms else list(cfg.forms)
    paths = args.paths.split(",")
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    n = len(cfg.spans)
    ms = tuple(kv.m for kv in disc.space.kvs)
    N = int(np.prod(ms))
    lattice = build_sampling_lattice(disc.space.kvs, cfg.M)
    # per call: equal plane slabs for the full assembly, cost-weighted plane slabs for the surrogate
    # (its box-boundary quadrature layers make the outer slabs heavy)
    from paper_1904_06971_b200.slabs import job_slabs

    slabs = {(f, path): job_slabs(ms, cfg.p, world, path, f, lattice.indices)[rank if world > 1 else 0]
             for f in (args.forms.split(",") if args.forms else list(cfg.forms)) for path in args.paths.split(",")}
    tilde = tilde_domain(cfg.p, ms)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    jobs = [(f, path) for f in forms for path in paths]
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
                                          tilde=tilde)
            n_irows = int(st.n_interp_rows)
        ms_, nl = _lib.last_timing()
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
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0.record(stream)
    nnz_tot = 0
    launches = 0
    ktimes = {}
    per_job = {}
    checks = np.zeros(5)
    for _ in range(args.steps):
        for f, path in jobs:
            nnz, nrows, nl, kt, cs, n_irows = one(f, path)
            nnz_tot += nnz
            launches += nl
            per_job[(f, path)] = (nnz, nrows, n_irows)
            for name, t in kt:
                key = (f, path, name)
                ktimes.setdefault(key, []).append(t)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms_dev = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    for f, path in jobs:  # untimed verification step: per-slab checksums, all-reduced over NCCL below
        checks += one(f, path, checksum=True)[4]
    if dist:
        t = torch.tensor([ms_dev], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_dev = float(t.item())
        tn = torch.tensor([float(nnz_tot)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tn)
        nnz_all = float(tn.item())
        tc = torch.tensor(checks, device="cuda", dtype=torch.float64)
        dist.all_reduce(tc)  # NCCL checksum all-reduce over the slabs
        checks = tc.cpu().numpy()
    else:
        nnz_all = float(nnz_tot)
    value = nnz_all / (ms_dev / 1e3)

    # ---- roofline of the dominant kernel (largest total device time)
    hbm, hbm_src = _peaks()
    g = disc.gauss
    E = int(np.prod(cfg.spans))
    plans = {}
    rows = []
    for (f, path, name), ts in ktimes.items():
        avg = sum(ts) / len(ts)
        nnz, nrows, n_irows = per_job[(f, path)]
        if name in ("assemble_tiles", "assemble_mma"):
            if path == "full":
                flops = f_elem(f, n, cfg.p, g) * E
            else:
                if f not in plans:
                    plans[f] = surrogate_plan(disc, pkg.ConstantSampling(cfg.M), cfg.q)
                flops = f_elem(f, n, cfg.p, g) * plans[f].active_elements
            if world > 1:
                flops = flops / world
            ach = flops / (avg / 1e3) / 1e12
            issued = 512.0 * dmma.get((f, path), 0)  # DMMA m8n8k4 f64 = 256 FMA
            rows.append({"kernel": f"{name}[{f},{path}]", "bound": "tensor", "achieved": ach,
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / FP64_PEAK_TFLOPS,
                         "issued_tflops": issued / (avg / 1e3) / 1e12 if issued else None,
                         "issued_frac": issued / (avg / 1e3) / 1e12 / FP64_PEAK_TFLOPS if issued else None,
                         "ms": avg, "flops": flops, "share": sum(ts)})
        elif name == "geom_D":
            rows.append({"kernel": f"geom_D[{f},{path}]", "bound": None, "ms": avg, "share": sum(ts)})
        elif name in ("interp_tiles", "interp_rows3"):
            # the kernel's own output: value + column of every slot of the interpolated rows
            b = 12 * n_irows * (2 * cfg.p + 1) ** n
            ach = b / (avg / 1e3) / 1e9
            rows.append({"kernel": f"{name}[{f}]", "bound": "hbm", "achieved": ach, "peak": hbm,
                         "unit": "GB/s", "frac": ach / hbm, "ms": avg, "bytes": b, "share": sum(ts)})
        elif name == "interp_slow_rows":
            rows.append({"kernel": f"interp_slow_rows[{f}]", "bound": None, "ms": avg, "share": sum(ts)})
    total_k = sum(sum(ts) for ts in ktimes.values())
    rows.sort(key=lambda r: -r["share"])
    for r in rows:
        r["share"] = r["share"] / total_k if total_k else None
    ranked = [r for r in rows if r.get("bound")]
    dom = dict(ranked[0]) if ranked else {}
    roof = {k: dom.get(k) for k in ("bound", "achieved", "peak", "unit", "frac", "issued_tflops", "issued_frac")}
    traffic = None
    try:  # DRAM bytes of the dominant kernel from its committed ncu --set full capture (per launch)
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")))
        t = tr.get(dom.get("kernel") or "")
        if t and world == 1:
            traffic = {"bytes": t["dram_bytes_read"] + t["dram_bytes_write"], "read": t["dram_bytes_read"],
                       "write": t["dram_bytes_write"], "source": t["source"]}
    except (OSError, ValueError, KeyError):
        traffic = None
    roof.update({"traffic": traffic["bytes"] if traffic else None, "traffic_detail": traffic, "kernel": dom.get("kernel"), "peak_source": "measured fp64 microbenchmark"
                 if dom.get("unit") == "TFLOP/s" else hbm_src,
                 "algorithmic": "SURVEY §8d reference-algorithm flops (F_elem x elements); the kernel is sum-factorised",
                 "issued": "issued_tflops / issued_frac: the fp64 tensor-core work the kernel actually executed "
                           "(counted DMMA instructions x 512 flops) against the same peak"})

    # ---- end to end through the public API (host buffers, H2D inside, D2H of the CSR)
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        h2d = d2h = 0
        nnz_e = 0
        _lib.host_staging_init(torch.cuda.current_device())  # one-time pinned ring, outside the timed region

        def e2e_job(f, path):
            fk = pkg.FormKind(f)
            slab = slabs[(f, path)]
            if path == "full":
                res, _, _ = pkg.assemble_device(fk, disc, slab=slab)
            else:
                mode = pkg.surrogate.DEFAULT_MODE[f].value
                res, _, _ = surrogate_device(fk, disc, cfg.M, cfg.q, mode, slab=slab, lattice=lattice, tilde=tilde)
            ip, ix, dd = res.to_host()
            res.free()
            return dd.size, ip.nbytes + ix.nbytes + dd.nbytes, _h2d_bytes(disc, path, lattice)

        def e2e_step():
            outs = [e2e_job(f, path) for f, path in jobs]
            return tuple(sum(o[i] for o in outs) for i in range(3))

        for _ in range(3):  # untimed warm-up (host result buffers mapped and pinned, as in any repeated assembly)
            e2e_step()
        _lib.host_pool_sync()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
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
        e2e = {"value": nnz_e / t_e2e, "unit": "nnz/s", "h2d_bytes_per_step": int(h2d // e2e_steps),
               "d2h_bytes_per_step": int(d2h // e2e_steps), "steps": e2e_steps,
               "api": "assemble_device/surrogate_device + Result.to_host (the calls behind assemble / build_surrogate_matrix)"}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, forms, paths, budget_s=args.cpu_budget)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_dev / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic geometry)",
            "config": {"workload": f"config{cfg.idx}:{cfg.name}", "forms": forms, "paths": paths, "p": cfg.p,
                       "spans": list(cfg.spans), "M": cfg.M, "q": cfg.q, "N": N,
                       "nnz_per_matrix": per_job[jobs[0]][0] if world == 1 else None,
                       "parallelism": f"row-slab x{world}" if world > 1 else "single GPU",
                       "l2": "outputs (8.9 GB/matrix at config 5) exceed L2; no flush needed"},
            "roofline": roof, "kernels": rows, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "checksum": {"nnz": checks[0], "sum": checks[1], "sumsq": checks[2]},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


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
# CPU baseline: the reference itself (baseline/_ref) when installed, else the oracle port
# ---------------------------------------------------------------------------------------------

def _cpu_sample(cfg):
    # bounded sample of the same workload: same geometry/form/p/q/M on a coarser mesh
    return {1: (32, 32), 2: (96, 96), 3: (14, 14, 14), 4: (128, 128), 5: (12, 12, 12)}[cfg.idx]


def _cpu_job(job):
    """One matrix of the CPU sample; runs in a worker process (single-threaded numpy)."""
    cfg_idx, f, path, use_ref = job
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.configs import CONFIGS

    cfg = CONFIGS[cfg_idx]
    spans = _cpu_sample(cfg)
    geom = cfg.geom()
    if use_ref:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        from surriga.assembly import FormKind, assemble, make_discretization
        from surriga.geometry import GeometryMap
        from surriga.bspline import NurbsWeights, make_tensor_space
        from surriga.surrogate import ConstantSampling, build_surrogate_matrix

        rg = GeometryMap(space=make_tensor_space(geom.space.p, geom.space.shape),
                         weights=NurbsWeights(geom.weights.weights, polynomial_weight=geom.weights.polynomial_weight),
                         control=geom.control)
        disc = make_discretization(rg, cfg.p, spans)
        fk = FormKind(f)
        t0 = time.perf_counter()
        if path == "full":
            A = assemble(fk, disc)
        else:
            A, _ = build_surrogate_matrix(fk, disc, ConstantSampling(cfg.M), q=cfg.q)
        return A.nnz, time.perf_counter() - t0
    from oracle import surriga_oracle as O

    disc = pkg.make_discretization(geom, cfg.p, spans)
    prob = O.problem_from_disc(pkg.FormKind(f), disc)
    t0 = time.perf_counter()
    if path == "full":
        _, ix, _, _, _ = O.assemble(prob)
    else:
        (_, ix, _), _, _ = O.surrogate(prob, cfg.M, cfg.q, None)
    return ix.size, time.perf_counter() - t0


def _have_ref():
    return os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "surriga"))


def _cpu_init(use_ref):
    """Worker start-up: single-threaded numpy, reference modules imported before the timed region."""
    os.environ["OMP_NUM_THREADS"] = "1"
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


def cpu_baseline(cfg, forms, paths, budget_s=60.0):
    """The reference's CPU path on every host core: the step's matrices (bounded sample mesh) are
    replicated over the cores, one single-threaded process per assembly (the reference assembly is
    serial numpy); value = all assembled nnz / wall time of the batch (pool start-up excluded)."""
    from concurrent.futures import ProcessPoolExecutor

    use_ref = _have_ref()
    cores = os.cpu_count() or 1
    base = [(cfg.idx, f, path, use_ref) for f in forms for path in paths]
    rep = max(1, cores // len(base))
    jobs = base * rep
    workers = max(1, min(len(jobs), cores))
    import multiprocessing as mp

    # spawn, not fork: the parent may hold a CUDA context and driver-pinned host buffers (a fork would
    # copy every pinned page into each child)
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"), initializer=_cpu_init,
                             initargs=(use_ref,)) as ex:
        list(ex.map(_cpu_warm, range(2 * workers)))
        t0 = time.perf_counter()
        res = list(ex.map(_cpu_job, jobs))
        wall = time.perf_counter() - t0
    nnz = sum(r[0] for r in res)
    return {"value": nnz / wall, "unit": "nnz/s", "cores": workers, "kind": "reference" if use_ref else "port",
            "sample": f"config {cfg.idx} workload ({', '.join(forms)} x {', '.join(paths)}) on a {_cpu_sample(cfg)} "
                      f"element mesh, {rep} copies of each matrix over {workers} single-threaded processes; "
                      f"{nnz} nnz in {wall:.1f} s",
            "per_matrix_s": [round(r[1], 3) for r in res[:len(base)]]}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1904_06971_b200.configs import CONFIGS

    cfg = CONFIGS[args.config]
    forms = args.forms.split(",") if args.forms else list(cfg.forms)
    paths = args.paths.split(",")
    for _ in range(args.warmup):
        pass  # the reference has no device state; warm-up = first import inside the workers
    vals = []
    last = None
    for _ in range(max(1, args.steps)):
        last = cpu_baseline(cfg, forms, paths)
        vals.append(last["value"])
    value = statistics.median(vals)
    cpu = dict(last)
    cpu["value"] = value
    line = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic geometry)", "impl": "reference",
            "config": {"workload": f"config{cfg.idx}:{cfg.name}", "forms": forms, "paths": paths},
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
    ap.add_argument("--cpu-budget", type=float, default=60.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
