#!/usr/bin/env python
"""Benchmark of the XDG solver hot path on B200 (contract: see DESIGN.md).

Default workload (BASELINE config 3, the config the metric's
"block-SpMV GB/s vs HBM peak" half is quoted on): the synthetic block-MSR
operator on 128^3 cells, p=2 (N=10), 7-point cell stencil, 5 % cut cells
with doubled species blocks, FP64; one step = one SpMV y = M x over the
whole operator (z-slab sharded with halo exchange when N > 1, strong
scaling).  Also reported in the same line: the XDG solves (DOF/s per solve,
the metric's first half) on the serialized reference hierarchies of
BASELINE config 1 (2D 16^2 p=2) and the 8^3 p=3 sphere case.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's CPU path (the oracle C restatement of
scipy csr_matvec over tocsr(), oracle/bsr_spmv.c, all host threads) on a
bounded sample of the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "XDG multigrid-GMRES DOF/s per solve; block-SpMV GB/s vs HBM peak"
NOMINAL_HBM_GBS = 8000.0


def ncu_traffic(kernel_substr: str = "spmv_warp_rows<10"):
    """dram read+write bytes per launch of the dominant kernel from the
    committed `ncu --set full` capture (profiles/), or None."""
    import csv

    path = os.path.join(ROOT, "profiles", "r2_spmv_ncu_raw.csv")
    try:
        rows = list(csv.reader(open(path)))
        h, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows[2:]:
            if kernel_substr in r[h.index("Kernel Name")]:
                tot = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    i = h.index(m)
                    tot += float(r[i]) * scale[units[i]]
                return tot
    except Exception:  # noqa: BLE001
        return None
    return None


def measured_peak():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        try:
            d = json.load(open(p))
            return float(d["hbm_gbs"]), "measured"
        except Exception:  # noqa: BLE001
            pass
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled DURING the timed region (B200_PROFILING.md)

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [v.strip() for v in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_spmv_sample(n_sample: int, seconds: float, threads: int):
    """Oracle C SpMV (restated scipy csr_matvec) on a 5 %-cut n^3 sample."""
    from oracle import cfg3, spmv

    rp, col, val, x = cfg3.build(n_sample)
    nbr, N = len(rp) - 1, val.shape[1]
    nnzb = len(col)
    B = 8 * N * N * nnzb + 4 * nnzb + 4 * (nbr + 1) + 16 * nbr * N
    spmv.bsr_spmv(rp, col, val, x, threads)  # warm
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 3:
        t0 = time.perf_counter()
        spmv.bsr_spmv(rp, col, val, x, threads)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return dict(value=B / t / 1e9, unit="GB/s", cores=threads, kind="port",
                sample=f"cfg3 recipe at {n_sample}^3 ({nbr} block rows, {nnzb} blocks, "
                       f"{B / 1e9:.3f} GB/SpMV), median of {len(times)} SpMVs, "
                       f"oracle/bsr_spmv.c on {threads} host threads",
                seconds=t, reps=len(times))


def _ref_size(args) -> tuple:
    """Full workload size for the reference arm when the host can hold the
    BSR operator (12.4 GB at 128^3, ~3x that while the recipe builds it),
    else the bounded sample; returns (n, why)."""
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = 0
    need = 3.2 * 12.4e9 * (args.n / 128) ** 3
    if avail >= need:
        return args.n, f"full {args.n}^3 operator ({avail / 1e9:.0f} GB host RAM available)"
    return args.ref_sample, (f"bounded {args.ref_sample}^3 sample: the {args.n}^3 operator "
                             f"needs ~{need / 1e9:.0f} GB host RAM to build, "
                             f"{avail / 1e9:.0f} GB available")


def run_reference(args):
    """The reference's CPU path (oracle C restatement of scipy csr_matvec over
    tocsr(), all host threads) on the same workload: the full 128^3
    operator when host RAM allows (same_config), else a bounded sample;
    each of the K timed steps is a batch of SpMVs of >= 0.5 s; W untimed
    warm-up steps."""
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return
    from oracle import cfg3, spmv

    threads = spmv.max_threads()
    n_ref, why = _ref_size(args)
    rp, col, val, x = cfg3.build(n_ref)
    nbr, N, nnzb = len(rp) - 1, val.shape[1], len(col)
    B = 8 * N * N * nnzb + 4 * nnzb + 4 * (nbr + 1) + 16 * nbr * N
    t0 = time.perf_counter()
    spmv.bsr_spmv(rp, col, val, x, threads)
    one = time.perf_counter() - t0
    reps = max(1, int(0.5 / max(one, 1e-6)))
    for _ in range(args.warmup):
        for _ in range(reps):
            spmv.bsr_spmv(rp, col, val, x, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(reps):
            spmv.bsr_spmv(rp, col, val, x, threads)
    wall = time.perf_counter() - t0
    ms_per_step = 1e3 * wall / args.steps
    value = B * reps * args.steps / wall / 1e9
    same = n_ref == args.n
    sample = (f"cfg3 recipe at {n_ref}^3 ({nbr} block rows, {nnzb} blocks, "
              f"{B / 1e9:.3f} GB/SpMV; {why}); one step = {reps} SpMV(s); oracle/bsr_spmv.c "
              f"(scipy csr_matvec order) on {threads} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY 8(d) cfg3 recipe, seed 0)",
        "config": {"workload": (f"BASELINE cfg3: block-MSR SpMV {args.n}^3 cells, p=2 (N=10), "
                                f"5% cut, {nbr} block rows, {nnzb} blocks") if same else
                               (f"cfg3 block-MSR SpMV, bounded sample {n_ref}^3 of the "
                                f"{args.n}^3 operator"),
                   "N": 10, "cut_fraction": 0.05, "same_config": same},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

CFG2_META = {  # BASELINE config 2: 32^3, p=3, sphere r=0.6, mu 1/1000
    "name": "cfg2", "dim": 3, "cells": 32, "degree": 3, "num_levels": 3,
    "omg": {"tolerance": 1e-10, "max_iterations": 2000, "k_lo": 2, "rm_max_columns": 800,
            "num_levels": 3},
    "gmres": {"tolerance": 1e-10, "max_iterations": 10000, "k_lo": 2, "gmres_restart": 50}}


def oracle_cfg2_box_estimate(solver: str, iterations: int, dofs_raw: int):
    """cpu_baseline of a cfg2 solve row: the CPU oracle (reference-exact
    numpy/scipy restatement) timed on the GPU box's host by
    tools/time_oracle_cfg2.py (1 and 3 iterations, first one with the lazy
    factorizations), extrapolated to the GPU's iteration count."""
    path = os.path.join(ROOT, "tests", "golden", "oracle_cfg2_timing_box.json")
    if not os.path.exists(path):
        return None
    t = json.load(open(path))
    k = "omg" if solver == "omg" else "gmres"
    if f"{k}_1it_s" not in t or f"{k}_3it_s" not in t:
        return None
    first, per = t[f"{k}_1it_s"], (t[f"{k}_3it_s"] - t[f"{k}_1it_s"]) / 2
    est = first + max(iterations - 1, 0) * per
    return {"value": dofs_raw / est, "unit": "DOF/s", "cores": t.get("cores"), "kind": "port",
            "sample": (f"oracle/solvers_np.py on the GPU box host ({t.get('cpu')}), "
                       f"1 and 3 iterations timed ({first:.1f} s incl. lazy factorizations, "
                       f"{per:.2f} s/iteration), extrapolated to {iterations} iterations = "
                       f"{est:.0f} s; tests/golden/oracle_cfg2_timing_box.json "
                       f"(tools/time_oracle_cfg2.py)"),
            "seconds_extrapolated": est}


def reference_cfg2_estimate(solver: str, iterations: int):
    """The reference's cfg2 solve time extrapolated from a bounded run of
    the reference itself in the build container
    (tests/golden/time_reference_cfg2.py: 1 and 3 iterations, the first
    including the lazy factorizations inside its solve timer): first +
    (iterations - 1) x per-iteration.  A lower bound for OMG (its RM space
    grows to 800 columns later in the solve)."""
    path = os.path.join(ROOT, "tests", "golden", "reference_cfg2_timing.json")
    if not os.path.exists(path):
        return None
    t = json.load(open(path))
    k = "omg" if solver == "omg" else "gmres"
    if f"{k}_1it_s" not in t or f"{k}_3it_s" not in t:
        return None
    first, per = t[f"{k}_1it_s"], (t[f"{k}_3it_s"] - t[f"{k}_1it_s"]) / 2
    est = first + max(iterations - 1, 0) * per
    return {"seconds": est, "first_iteration_s": first, "per_iteration_s": per,
            "iterations": iterations, "cores": t.get("cores"),
            "where": "build container (reference cutdg, scipy/numpy)",
            "source": "tests/golden/reference_cfg2_timing.json"}


def native_cfg2(world: int = 1):
    """BASELINE config 2 built by this package's own setup pipeline
    (case.assemble_case: geometry, agglomeration, SIP assembly, hierarchy);
    returns (hierarchy, meta, setup row)."""
    from paper_2003_02431_b200.case import BenchCase, assemble_case

    c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
    case = BenchCase(dim=3, cells=32, degree=3, levelset="sphere",
                     levelset_params={"center": tuple(c), "radius": 0.6}, mu_a=1.0,
                     mu_b=1000.0, alpha=0.1, num_levels=3,
                     workers=max(1, (os.cpu_count() or 1) // world))
    t0 = time.perf_counter()
    asm = assemble_case(case)
    setup = time.perf_counter() - t0
    meta = dict(CFG2_META, dofs_raw=int(len(asm.rhs)))
    row = {"case": "cfg2", "what": "native setup (mesh, cut cells, agglomeration, SIP "
                                   "assembly, 3-level hierarchy)",
           "setup_s": setup, "phases": {k: round(v, 3) for k, v in asm.phase_times.items()},
           "dofs_raw": meta["dofs_raw"], "level_blocks": [
               asm.hierarchy.level(lam).data.num_blocks
               for lam in range(1, asm.hierarchy.num_levels + 1)],
           "reference_setup_s_build_container": 847.8,
           "reference_setup_source": "tests/golden/make_large.py cfg2 (cutdg assemble_case, "
                                     "1 host thread)"}
    return asm.hierarchy, meta, row


def ref_envelope(case, z, solver, meta):
    """[min, max] iterations of the reference under +-1-ulp perturbations of
    b: the K = 20-40 run envelope of {case}_env.npz at
    the solve's tolerance when present, else the fixture's K = 5 one."""
    tol = meta[solver].get("tolerance", 1e-10)
    p = os.path.join(ROOT, "tests", "golden", f"{case}_env.npz")
    key = f"{solver}_tol{tol:.0e}"
    if os.path.exists(p):
        e = np.load(p)
        if key in e.files:
            return {"min": int(e[key].min()), "max": int(e[key].max()), "runs": int(len(e[key]))}
    if f"{solver}_envelope" in z:
        e = z[f"{solver}_envelope"]
        return {"min": int(e.min()), "max": int(e.max()), "runs": int(len(e))}
    return None


def time_solves(torch, budget_s: float):
    """XDG solves: DOF/s per solve on the reference's serialized hierarchies
    (cfg1, 8^3 p=3 sphere, and the full-size cfg2 when its fixture is
    present) or on the natively built cfg2 hierarchy otherwise."""
    from paper_2003_02431_b200 import solvers as S
    from paper_2003_02431_b200.hierarchy import load_hierarchy
    from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve

    peak, peak_kind = measured_peak()
    # one-time process warm-up (kernel module loading) outside the timed
    # solves -- the reference's scipy/LAPACK is likewise already loaded
    from paper_2003_02431_b200.device import Context
    from paper_2003_02431_b200.factor import warmup

    warmup(Context.get())

    def cases():
        for case in ("cfg1", "sphere8p3", "large/s16p3"):
            path = os.path.join(ROOT, "tests", "golden", f"{case}.npz")
            if os.path.exists(path):
                z = np.load(path)
                yield case, z, json.loads(bytes(z["meta"]).decode()), load_hierarchy(z), None
        path = os.path.join(ROOT, "tests", "golden", "large", "cfg2.npz")
        if os.path.exists(path) and not os.environ.get("XDG_BENCH_NATIVE_CFG2"):
            z = np.load(path)
            meta = json.loads(bytes(z["meta"]).decode())
            meta["gmres"] = dict(meta["gmres"], max_iterations=CFG2_META["gmres"][
                "max_iterations"])
            yield "large/cfg2", z, meta, load_hierarchy(z), None
        else:
            hier, meta, row = native_cfg2()
            yield "cfg2 (native setup)", {}, meta, hier, row

    out = []
    t_start = time.perf_counter()
    for case, z, meta, hier, setup_row in cases():
        if setup_row is not None:
            out.append(setup_row)
        lv = hier.level(1)
        for solver in ("gmres", "omg"):
            if time.perf_counter() - t_start > budget_s:
                break
            cfg = SolverConfig(**meta[solver])
            torch.cuda.synchronize()
            try:
                if solver == "omg":
                    octx = S._OmgContext(cfg, 1)
                    x, rep = ortho_mg_solve(hier, lv.rhs, None, cfg, 1, octx)
                    loop = dict(octx.last_loop)
                else:
                    x, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=meta["dim"])
                    loop = dict(S.LAST_LOOP)
            except NotImplementedError as exc:
                out.append({"case": case, "solver": solver, "unsupported": str(exc)})
                continue
            if f"{solver}_x" in z:
                ref_x = z[f"{solver}_x"]
                rel = float(np.linalg.norm(x - ref_x) / np.linalg.norm(ref_x))
            else:  # large fixtures: no reference solve (hours on the CPU)
                rel = None
            ref_s = meta.get(f"{solver}_seconds")
            ref_extrap = None
            if case.endswith("cfg2") or case.startswith("cfg2"):
                ref_extrap = reference_cfg2_estimate(solver, rep.iterations)
            cpu_here, cpu_base = None, None
            if case == "cfg1":  # bounded: ~10 s of CPU per solver
                from oracle import solvers_np

                _, cpu_it, cpu_here = solvers_np.timed_solve(z, meta, solver)
                cpu_base = {"value": meta["dofs_raw"] / cpu_here, "unit": "DOF/s",
                            "cores": os.cpu_count(), "kind": "port",
                            "sample": (f"full cfg1 solve ({cpu_it} iterations) by "
                                       f"oracle/solvers_np.py on this host, timed live")}
            elif "cfg2" in case:
                cpu_base = oracle_cfg2_box_estimate(solver, rep.iterations, meta["dofs_raw"])
            out.append({
                "case": case, "solver": "omg" if solver == "omg" else "gmres-pmg",
                "config": meta[solver], "dofs_raw": meta["dofs_raw"],
                "dofs_agglomerated": lv.num_dofs, "iterations": rep.iterations,
                "ref_iterations_envelope": ref_envelope(case, z, solver, meta),
                "converged": rep.converged, "final_residual": rep.final_residual,
                "relative_residual": rep.final_residual / float(np.linalg.norm(lv.rhs)),
                "solve_s": rep.time_iterations,
                "dof_per_s": meta["dofs_raw"] / rep.time_iterations,
                "ms_per_iteration": 1e3 * rep.time_iterations / max(rep.iterations, 1),
                "setup_s": loop["setup_seconds"], "loop_s": loop["seconds"],
                "loop_algorithmic_bytes": loop["bytes"],
                "loop_GBs": loop["bytes"] / max(loop["seconds"], 1e-12) / 1e9,
                "loop_frac_of_hbm_peak": loop["bytes"] / max(loop["seconds"], 1e-12)
                / 1e9 / peak,
                "loop_frac_of_nominal_8TBs": loop["bytes"] / max(loop["seconds"], 1e-12)
                / 1e9 / NOMINAL_HBM_GBS,
                "rel_err_vs_reference": rel,
                "reference_cpu_s_build_container": ref_s,
                "cpu_oracle_s_this_host": cpu_here,
                "cpu_oracle_dof_per_s_this_host":
                    (meta["dofs_raw"] / cpu_here) if cpu_here else None,
                "cpu_oracle_cores": os.cpu_count(),
                "reference_cpu_dof_per_s_build_container":
                    (meta["dofs_raw"] / ref_s) if ref_s else None,
                "reference_cpu_extrapolated": ref_extrap,
                "cpu_baseline": cpu_base,
            })
    return out


def time_matops(torch):
    """The paper's Table-2 instance (6^3 cells, k=5, benchmark surface): SpMV
    and the Galerkin product R0^T M R0 (micro_bench_matops, bench.py:326-352),
    next to the published BoSSS numbers and the
    reference timings recorded when the fixture was generated."""
    from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout
    from paper_2003_02431_b200.hierarchy import fixture_array
    from paper_2003_02431_b200.transfer import galerkin_device, galerkin_restrict

    path = os.path.join(ROOT, "tests", "golden", "large", "matops_6_k5.npz")
    if not os.path.exists(path):
        return {"skipped": "tests/golden/large/matops_6_k5.npz absent"}
    z = np.load(path)

    def mat(prefix):
        rp = z[prefix + "_row_ptr"]
        val = fixture_array(z, prefix + "_val")
        N = val.shape[1]
        return BlockSparseMatrix.from_bsr(rp, z[prefix + "_col"], val,
                                          uniform_layout(len(rp) - 1, N),
                                          uniform_layout(int(z[prefix + "_ncols"]), N))

    M, R0 = mat("M"), mat("R0")
    D = M.device()
    v = torch.ones(D.nbc * D.N, dtype=torch.float64, device="cuda")
    y = D.spmv(v)

    def events(fn, reps):
        ts = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        return statistics.median(ts)

    events(lambda: D.spmv(v, y), 3)
    spmv_ms = events(lambda: D.spmv(v, y), 20)
    galerkin_device(M, R0)
    gal_dev_ms = events(lambda: galerkin_device(M, R0), 5)
    t0 = time.perf_counter()
    galerkin_restrict(M, None, R0)
    gal_api_ms = 1e3 * (time.perf_counter() - t0)
    return {"instance": "6^3 cells, k=5 (N=56), paper benchmark surface",
            "nonzero_rows": int(z["nonzero_rows"]),
            "matvec_ms": spmv_ms, "matvec_GBs": D.algorithmic_bytes() / spmv_ms / 1e6,
            "matmat_device_ms": gal_dev_ms, "matmat_api_ms": gal_api_ms,
            "reference_cpu_build_container_ms": {"matvec": float(z["matvec_ms"]),
                                                 "matmat": float(z["matmat_ms"])},
            "published_bosss_ms": {"matvec_1core_i7": 14.6, "matvec_4core_i7": 8.99,
                                   "matmat_1core_i7": 3880.0, "matmat_4core_i7": 1293.0,
                                   "source": "PAPER.md:1328-1338 (24,192 rows)"}}


def time_dist_solve(torch, dist):
    """Distributed OMG (z-ordered row partition per level, NCCL) on the
    serialized full-size BASELINE config-2 hierarchy, if present."""
    from paper_2003_02431_b200.dist_solvers import dist_ortho_mg_solve
    from paper_2003_02431_b200.hierarchy import load_hierarchy
    from paper_2003_02431_b200.solvers import SolverConfig

    path = os.path.join(ROOT, "tests", "golden", "large", "cfg2.npz")
    if os.path.exists(path):
        z = np.load(path)
        meta = json.loads(bytes(z["meta"]).decode())
        hier = load_hierarchy(z)
    else:  # every rank builds the hierarchy with its share of the host cores
        hier, meta, _ = native_cfg2(dist.get_world_size())
    dist.barrier()
    x, (r0, r1), rep = dist_ortho_mg_solve(hier, np.asarray(hier.level(1).rhs),
                                           SolverConfig(**meta["omg"]))
    t = torch.tensor([rep.time_iterations], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"case": "large/cfg2", "solver": "omg (distributed)", "n_gpus": dist.get_world_size(),
            "dofs_raw": meta["dofs_raw"], "iterations": rep.iterations,
            "converged": rep.converged, "solve_s": float(t.item()),
            "dof_per_s": meta["dofs_raw"] / float(t.item())}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; "
                         f"run without torchrun to let bench.py spawn the ranks")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2003_02431_b200 import _native as nat
    from paper_2003_02431_b200.device import Context
    from paper_2003_02431_b200.distributed import DistributedSpMV, HaloPlan
    from paper_2003_02431_b200.synthetic import cfg3_slab_device

    ctx = Context.get(dev)
    t_setup = time.perf_counter()
    s = cfg3_slab_device(args.n, rank, world, ctx=ctx)
    D = s["D"]
    N = D.N
    nloc = s["row1"] - s["row0"]
    ghosts = np.concatenate([s["halo_lo"], s["halo_hi"]])
    # global row partition
    starts = torch.zeros(world + 1, dtype=torch.int64)
    if world > 1:
        r0 = torch.tensor([s["row0"]], dtype=torch.int64, device=dev)
        allr = [torch.zeros_like(r0) for _ in range(world)]
        dist.all_gather(allr, r0)
        starts[:world] = torch.cat(allr).cpu()
    starts[world] = s["nbr_global"]
    halo = HaloPlan(starts.numpy(), ghosts, rank, world, N, dev)
    op = DistributedSpMV(D, halo)
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    x_ext = torch.randn((nloc + len(ghosts)) * N, generator=g, device=dev, dtype=torch.float64)
    y = torch.empty(nloc * N, dtype=torch.float64, device=dev)
    setup_s = time.perf_counter() - t_setup

    # algorithmic bytes of the whole operator and of this rank
    nnzb_g = int(D.nnzb)
    if world > 1:
        t = torch.tensor([D.nnzb], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        nnzb_g = int(t.item())
    nbr_g = s["nbr_global"]
    B_global = 8 * N * N * nnzb_g + 4 * nnzb_g + 4 * (nbr_g + 1) + 16 * nbr_g * N
    B_local = D.algorithmic_bytes()

    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        op(x_ext, y)
    barrier()
    # timed region: K steps; per-step kernel events for the roofline
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        start.record(stream)
        for k in range(args.steps):
            ev[k][0].record(stream)
            op(x_ext, y)
            ev[k][1].record(stream)
        end.record(stream)
        barrier()
    elapsed_ms = start.elapsed_time(end)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = B_global * args.steps / (elapsed_ms * 1e-3) / 1e9
    # dominant kernel: the SpMV launch(es) of one step (N=1: one launch)
    kern_ms = statistics.mean(step_ms)
    achieved = B_local / (kern_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peak()
    gpu_launches = args.steps * ((1 if world == 1 else 3) + (len(halo.sends) if world > 1 else 0))

    # ---- e2e through the C-ABI with pinned host buffers -------------------
    xh = torch.empty(nloc * N, dtype=torch.float64, pin_memory=True)
    xh.copy_(x_ext[: nloc * N].cpu())
    yh = torch.empty(nloc * N, dtype=torch.float64, pin_memory=True)
    xd = x_ext  # device buffer the host copy lands in
    if world == 1:
        # the public drop-in call on host buffers: BlockSparseMatrix.matvec
        # (blockmatrix.py:119-125 analogue) with pinned x / out -> pinned
        # staging-free HostStreamSpMV (z-slab chunks: H2D || xdg_bsr_spmv
        # per chunk through the C-ABI || D2H), blocking until y has landed
        from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout

        Mpub = BlockSparseMatrix.from_device(D, uniform_layout(nloc, N),
                                             uniform_layout(D.nbc, N))
        Mpub.matvec(xh, out=yh)
        op(x_ext, y)
        torch.cuda.synchronize(dev)
        e2e_exact = bool(torch.equal(yh, y.cpu()))
        step = (lambda: Mpub.matvec(xh, out=yh))
        nchunks = len(Mpub._host_streamer(D)[0].bounds) - 1
        e2e_path = (f"BlockSparseMatrix.matvec(pinned x, out=pinned y): H2D ({nchunks} z-slab "
                    "chunks) || xdg_bsr_spmv per chunk (C-ABI) || D2H y, full-duplex "
                    "overlapped, host-synchronous per call")
    else:
        def step():
            xd[: nloc * N].copy_(xh, non_blocking=True)
            op(xd, y)
            yh.copy_(y, non_blocking=True)
        e2e_exact, e2e_path = None, "pinned host x -> H2D -> halo SpMV (C-ABI) -> D2H y"
    for _ in range(2):
        step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    extra_e2e = {}
    if world == 1:
        # (a) the same products enqueued back to back (sync=False: the next
        # product's H2D overlaps this one's D2H); (b) numpy in -> numpy out
        # (the reference's exact contract: + pinned staging copies)
        hs = Mpub._host_stream[0]
        for _ in range(2):
            hs(xh, yh, sync=False)
        hs.wait()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            hs(xh, yh, sync=False)
        hs.wait()
        e1.record(stream)
        barrier()
        ov_ms = e0.elapsed_time(e1)
        xnp = xh.numpy().copy()
        Mpub.matvec(xnp)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ynp = Mpub.matvec(xnp)
        np_s = time.perf_counter() - t0
        extra_e2e = {
            "overlapped_back_to_back": {
                "value": B_global * args.steps / (ov_ms * 1e-3) / 1e9, "unit": "GB/s",
                "what": "HostStreamSpMV(sync=False) products enqueued back to back"},
            "numpy_in_numpy_out": {
                "value": B_global * args.steps / np_s / 1e9, "unit": "GB/s",
                "what": "BlockSparseMatrix.matvec(numpy x) -> numpy y (pinned staging "
                        "copies included), host wall clock",
                "bit_identical": bool(np.array_equal(ynp, yh.numpy()))}}
    # the e2e roofline: the same bytes as raw concurrent pinned H2D + D2H
    # copies (PCIe full duplex), no compute
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    yd_raw = torch.empty_like(y)
    for rep in range(2):
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        s1.wait_stream(stream)
        s2.wait_stream(stream)
        for _ in range(args.steps):
            with torch.cuda.stream(s1):
                yd_raw.copy_(xh, non_blocking=True)
            with torch.cuda.stream(s2):
                yh.copy_(y, non_blocking=True)
        stream.wait_stream(s1)
        stream.wait_stream(s2)
        f1.record(stream)
        f1.synchronize()
    pcie_ms = f0.elapsed_time(f1)
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    e2e_val = B_global * args.steps / (e2e_ms * 1e-3) / 1e9

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (SURVEY 8(d) cfg3 recipe pattern, seed 0; "
                                    "seeded device values of the recipe's distributions)",
            "config": {"workload": f"BASELINE cfg3: block-MSR SpMV {args.n}^3 cells, p=2 "
                                   f"(N=10), 5% cut, {nbr_g} block rows, {nnzb_g} blocks",
                       "algorithmic_bytes_per_step": B_global,
                       "l2": "inputs larger than L2 (matrix 12.4 GB >> 126 MB); no flush",
                       "parallelism": f"z-slab x{world}, NCCL halo" if world > 1 else "1 GPU",
                       "setup_s": setup_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "frac_of_nominal_8TBs": achieved / NOMINAL_HBM_GBS,
                         "kernel": "xdg spmv_warp_rows<10>",
                         "kernel_ms": kern_ms, "bytes_per_launch": B_local,
                         "traffic": ncu_traffic() if args.n == 128 and world == 1 else None,
                         "traffic_source": "profiles/r2_spmv_ncu_raw.csv (ncu --set full, "
                                           "same command, dram__bytes_read+write per launch)"},
            "e2e": {"value": e2e_val, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * nloc * N, "d2h_bytes_per_step": 8 * nloc * N,
                    "path": e2e_path, "bit_identical_to_device_spmv": e2e_exact,
                    "pcie_duplex_floor": {
                        "value": B_global * args.steps / (pcie_ms * 1e-3) / 1e9,
                        "unit": "GB/s", "what": "the step's H2D + D2H bytes as raw "
                                                "concurrent pinned copies, no compute"},
                    "frac_of_pcie_floor": pcie_ms / e2e_ms, **extra_e2e},
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
    if world == 1 and not args.no_solve:
        try:
            line["solve"] = time_solves(torch, args.solve_budget)
        except Exception as exc:  # noqa: BLE001
            line["solve_error"] = repr(exc)
        try:
            line["matops"] = time_matops(torch)
        except Exception as exc:  # noqa: BLE001
            line["matops"] = {"error": repr(exc)}
    if world > 1 and not args.no_solve:
        # DOF/s of the full-size cfg2 OMG solve over all ranks (dist_solvers)
        try:
            solve = time_dist_solve(torch, dist)
        except Exception as exc:  # noqa: BLE001
            solve = {"error": repr(exc)}
        if rank == 0:
            line["solve"] = [solve]
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import spmv as ospmv

            line["cpu_baseline"] = {k: v for k, v in cpu_spmv_sample(
                args.ref_sample, args.cpu_seconds, ospmv.max_threads()).items()
                if k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    del nat


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: launch N ranks (one
    process per GPU, NCCL) through torch.distributed.run on 127.0.0.1 with
    the same arguments; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--ref-sample", type=int, default=48)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--solve-budget", type=float, default=240.0)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
