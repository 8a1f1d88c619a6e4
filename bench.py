"""Benchmark of the B200 MG-GMRES / Vanka linear-solve path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload 3d_large]

One step = one full right-preconditioned GMRES solve to 1e-8 of the seeded
condensed velocity-pressure Jacobian (BASELINE config 3: 3D, 128x32x32 Q2
hexahedra, 5 levels, ~4.3M FP64 dofs, 108x108 Vanka patch inverses), with
the level hierarchy and patch inverses resident in HBM.  ``value`` is
solves/s over all ranks with the RHS already on the device; ``e2e`` is the
same through the public ``DeviceMgSolver.gmres`` call from pinned host
buffers (H2D of b and D2H of x inside the timed region).  N>1 runs
independent replicas (the path does not shard).

``--impl reference`` runs the UNMODIFIED reference package (pure Python,
installed into ``baseline/_ref``, which travels to the GPU box) through its
own API (``baseline/ref_arm.py``): its own problem setup and assembly, then
complete ``gmres`` + ``MgSolver`` solves on the box's host cores (all
threads), timing as many solves as fit in ``--ref-budget-s`` and reporting
the number actually timed.  It never imports the product package.

Both arms refuse to print a line whose solve does not reproduce the
committed golden history (``check_against_golden``).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MG-GMRES solves/s and Vanka sweeps/s (FP64) at 3D 4.3M dofs; % of HBM roofline"
UNIT = "solves/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------- parity gate
class ParityError(RuntimeError):
    """The solve about to be timed does not reproduce the committed golden."""


GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def golden_for(workload):
    """Committed golden of a workload's full-size solve: the reference's own
    run (tests/golden/<w>.json) where the reference could run it, else the
    pinned CPU oracle's (tests/golden/<w>_oracle.json)."""
    for name in (f"{workload}.json", f"{workload}_oracle.json"):
        path = os.path.join(GOLDEN_DIR, name)
        if os.path.exists(path):
            with open(path) as f:
                g = json.load(f)
            if "residuals" in g:
                return path, g
    return None, None


def check_against_golden(workload, iterations, residuals, x_checksums,
                         hist_tol=1e-10, x_tol=1e-9):
    """north_star's parity bar on the solve bench.py times: identical
    iteration count, residual history within 1e-10 relative, solution
    checksums within 1e-9.  Raises ParityError otherwise."""
    path, g = golden_for(workload)
    if g is None:
        raise ParityError(f"no committed golden history for workload {workload}")
    rel = os.path.relpath(path, ROOT)
    if iterations != g["iterations"] or len(residuals) != len(g["residuals"]):
        raise ParityError(f"{workload}: {iterations} GMRES iterations, golden {rel} has "
                          f"{g['iterations']}")
    r, rr = np.asarray(residuals, dtype=float), np.asarray(g["residuals"], dtype=float)
    hist = float(np.max(np.abs(r - rr) / rr))
    if not hist < hist_tol:
        raise ParityError(f"{workload}: residual history differs from {rel} by {hist:.3e}")
    xrel = None
    if x_checksums is not None:
        c, cc = np.asarray(x_checksums), np.asarray(g["x_checksums"])
        xrel = float(np.max(np.abs(c - cc) / np.abs(cc)))
        if not xrel <= x_tol:
            raise ParityError(f"{workload}: solution checksums differ from {rel} by {xrel:.3e}")
    return {"source": rel, "iterations": int(g["iterations"]),
            "max_rel_history_diff": hist, "max_rel_checksum_diff": xrel}


def vector_checksums(x):
    """tests/golden_util.vector_checksums (norm + two seeded projections)."""
    rng = np.random.default_rng(99)
    ps = [rng.standard_normal(len(x)) for _ in range(2)]
    return [float(np.linalg.norm(x))] + [float(p @ x) for p in ps]


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML from
    a background thread every 10 ms (so that a 0.1 s timed region of the small
    workloads still yields ~10 samples), else `nvidia-smi -lms 200`."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.thread = None
        self.lines = []

    def _nvml_loop(self, nv, handle, stop):
        names = [("hw_slowdown", nv.nvmlClocksEventReasonHwSlowdown),
                 ("hw_thermal_slowdown", nv.nvmlClocksEventReasonHwThermalSlowdown),
                 ("sw_thermal_slowdown", nv.nvmlClocksEventReasonSwThermalSlowdown),
                 ("sw_power_cap", nv.nvmlClocksEventReasonSwPowerCap)]
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(handle, nv.NVML_CLOCK_SM)
        except Exception:
            mx = 0
        while not stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(handle, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(handle)
                self.lines.append(",".join([str(sm), str(mx)] + [
                    "Active" if mask & bit else "Not Active" for _, bit in names]))
            except Exception:
                break
            stop.wait(0.01)

    def __enter__(self):
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            # NVML enumerates all boards: map the CUDA device through its PCI bus id
            import torch
            bus = torch.cuda.get_device_properties(self.index).pci_bus_id \
                if hasattr(torch.cuda.get_device_properties(self.index), "pci_bus_id") else None
            handle = None
            if bus is not None:
                for i in range(nv.nvmlDeviceGetCount()):
                    h = nv.nvmlDeviceGetHandleByIndex(i)
                    if nv.nvmlDeviceGetPciInfo(h).bus == bus:
                        handle = h
                        break
            if handle is None:
                visible = os.environ.get("CUDA_VISIBLE_DEVICES", "")
                ids = [v for v in visible.split(",") if v.strip().isdigit()]
                phys = int(ids[self.index]) if self.index < len(ids) else self.index
                handle = nv.nvmlDeviceGetHandleByIndex(phys)
            nv.nvmlDeviceGetClockInfo(handle, nv.NVML_CLOCK_SM)
            nv.nvmlDeviceGetCurrentClocksEventReasons(handle)
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._nvml_loop,
                                           args=(nv, handle, self.stop), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=2)
            return
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        src = "nvml, 10 ms" if self.thread is not None else "nvidia-smi -lms 200"
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "sampler": src}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm), "sampler": src}


def max_over_ranks(values, world, device=None):
    """Element-wise max of per-rank timings (replicas: the slowest rank sets
    the whole-job time)."""
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def whole_job_rate(units_per_rank, world, ms):
    """Units processed by all ranks / max-over-ranks time."""
    return world * units_per_rank / (ms * 1e-3)


# ------------------------------------------------------------------------ algorithmic bytes
def host_case_from_device(wl, prob, solver, b):
    """Host copies of the device-assembled operators (CPU baseline input)."""
    from paper_1904_02401_b200 import fem, workloads as W
    mats = []
    for l, lvl in enumerate(prob.levels):
        data, pp = solver.matrix_data(l, lvl.pattern)
        mats.append(fem.SplitBlockMatrix(lvl.pattern, data, pp))
    return W.Case(wl, prob, None, None, mats, solver.patches, [None] * len(mats),
                  solver.prolongations, b)


def kernel_bytes(case, wl):
    """Algorithmic HBM bytes of one finest-level launch of each kernel."""
    p = case.problem.levels[-1].pattern
    nc = wl.dim + 1
    n = p.n_nodes * nc
    spmv = (p.nnzb * (nc * nc * 8 + 4) + (p.n_nodes + 1) * 8 + p.nnz_pp * 12
            + ((p.n_nodes + 1) * 8 if p.nnz_pp else 0) + 3 * n * 8)
    vanka = 0
    for g, _ in case.patches[-1].groups:
        npd = g.shape[1] * nc
        vanka += len(g) * (npd * npd * 8 + npd * 8 + g.shape[1] * 4)
    vanka += n * 8
    return {"spmv": spmv, "vanka_apply": vanka}


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, world):
    import torch
    from paper_1904_02401_b200 import device, workloads as W
    wl = W.CONFIGS[args.workload]
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    prob, solver, b, setup = W.build_device_solver(wl, stream=stream.cuda_stream,
                                                   use_graph=not args.no_graph)
    torch.cuda.synchronize()
    t_setup_total = time.perf_counter() - t0
    case = W.Case(wl, prob, None, None, [], solver.patches, [], solver.prolongations, b)
    solver.reserve(wl.max_iter)
    log(f"[rank {rank}] setup {t_setup_total:.1f}s {setup}")
    # warm re-assembly + Vanka/coarse re-factorisation (what every Newton
    # reassembly costs; the first call above also pays lazy module loading)
    U, Up = W.linearisation_state(wl, prob)
    t0 = time.perf_counter()
    for l, lvl in enumerate(prob.levels):
        solver.asm_momentum(l, lvl, prob.mats, wl.dt, wl.theta, prob.restrict_state(U, l),
                            prob.restrict_state(Up, l))
    # the launch stream only: the coarse inverse started by the level-0
    # assembly keeps running on the library's side stream and is joined by
    # factorize()
    torch.cuda.current_stream().synchronize()
    t1 = time.perf_counter()
    solver.factorize()
    torch.cuda.synchronize()
    setup["warm_device_assembly"] = t1 - t0
    setup["warm_vanka_setup"] = time.perf_counter() - t1
    for lvl in prob.levels:          # host geometry tables are not needed any more
        lvl.G = None                 # (keeps N replicas' host memory in check)
    b_dev = torch.from_numpy(case.b).to(dev)
    x_dev = torch.empty_like(b_dev)

    def solve():
        return solver.gmres(b_dev, rel_tol=wl.rel_tol, max_iter=wl.max_iter, x_out=x_dev)

    for _ in range(args.warmup):
        _, st = solve()
    iterations = st.iterations
    log(f"[rank {rank}] warm-up done: {iterations} GMRES iterations")
    # parity gate: the solve about to be timed must reproduce the golden
    parity = check_against_golden(args.workload, st.iterations, st.residuals,
                                  vector_checksums(x_dev.cpu().numpy()))
    log(f"[rank {rank}] parity vs {parity['source']}: history {parity['max_rel_history_diff']:.1e}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- timed region: device-resident RHS, V-cycle replayed as a CUDA graph
    launches0 = solver.kernel_launches()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            _, st = solve()
        ev1.record(stream)
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    launches = solver.kernel_launches() - launches0
    if not st.converged or st.iterations != iterations:
        raise RuntimeError("timed solves diverged from the warm-up solves")

    # ---- instrumented pass: the same K solves with a CUDA-event pair around
    # every kernel on the launch stream (graph replay off while recording)
    solver.profile(True)
    solver.profile_read(reset=True)
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        solve()
    ev1.record(stream)
    barrier()
    ms_prof = ev0.elapsed_time(ev1)
    prof = solver.profile_read(reset=True)
    solver.profile(False)

    # ---- end to end through the public API from pinned host buffers
    b_host = torch.from_numpy(case.b).pin_memory().numpy()
    x_host = torch.empty(len(case.b), dtype=torch.float64).pin_memory().numpy()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        solver.gmres(b_host, rel_tol=wl.rel_tol, max_iter=wl.max_iter, x_out=x_host)
    e1.record(stream)
    barrier()
    ms_e2e = e0.elapsed_time(e1)

    # ---- standalone finest-level sweep and SpMV throughput
    L = solver.n_levels - 1
    xs = torch.zeros_like(b_dev)
    nsw = args.sweeps
    for _ in range(3):
        solver.sweep(L, xs, b_dev)
    barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(nsw):
        solver.sweep(L, xs, b_dev)
    s1.record(stream)
    barrier()
    ms_sweep = s0.elapsed_time(s1) / nsw
    y = torch.empty_like(b_dev)
    s0.record(stream)
    for _ in range(nsw):
        solver.spmv(L, xs, None, y)
    s1.record(stream)
    barrier()
    ms_spmv = s0.elapsed_time(s1) / nsw

    # ---- max over ranks
    ms_total, ms_e2e, ms_sweep, ms_spmv = max_over_ranks(
        [ms_total, ms_e2e, ms_sweep, ms_spmv], world, dev)
    if rank != 0:
        return None

    kb = kernel_bytes(case, wl)
    n = len(case.b)
    info = WORKLOADS[args.workload]
    if n != info["dofs"] or kb["spmv"] + kb["vanka_apply"] != info["sweep_bytes"]:
        raise RuntimeError(f"workload table out of date for {args.workload}")
    peak, peak_src = peaks()
    kernels = {}
    total_prof = sum(v[1] for v in prof.values())
    for (kind, finest), (cnt, ms) in prof.items():
        if cnt:
            key = f"{kind}{'_finest' if finest else '_coarser'}"
            kernels[key] = {"launches": cnt, "avg_ms": ms / cnt, "share": ms / ms_prof}
    # per-application figures: the library records one event pair around a
    # whole Vanka application (one launch per run of same-size patch groups:
    # fluid + solid 108x108 share one, the 500x500 macros get their own);
    # kb counts the bytes of all groups
    dom = max(("spmv", "vanka_apply"), key=lambda k: prof[(k, True)][1])
    cnt, ms = prof[(dom, True)]
    avg_ms = ms / cnt
    achieved = kb[dom] / (avg_ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.workload, dom)
    n = len(case.b)
    solves_per_s = whole_job_rate(args.steps, world, ms_total)
    out = {
        "metric": METRIC, "value": solves_per_s, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded sine-mode linearisation state and RHS, workload {args.workload})",
        "config": workload_config(args.workload, iterations, world),
        "parity": parity,
        "e2e": {"value": world * args.steps / (ms_e2e * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * 8 + 8 * (iterations + 1)},
        "gpu_launches": launches,
        "algorithmic_bytes": kb,
        "roofline": {"bound": "hbm", "kernel": f"{dom} (finest level)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algorithmic_bytes_per_launch": kb[dom],
                     "avg_launch_ms": avg_ms, "share_of_step": ms / ms_prof,
                     "peak_source": peak_src},
        "vanka_sweeps_per_s": 1e3 / ms_sweep,
        "vanka_sweeps_timed": nsw,      # standalone finest-level sweep benchmark (--sweeps)
        "vanka_sweep_ms": ms_sweep,
        "spmv_ms": ms_spmv, "spmv_gbs": kb["spmv"] / (ms_spmv * 1e-3) / 1e9,
        "vanka_apply_gbs": kb["vanka_apply"] / (prof[("vanka_apply", True)][1] /
                                                 max(1, prof[("vanka_apply", True)][0]) * 1e-3) / 1e9,
        "spmv_in_solve_gbs": kb["spmv"] / (prof[("spmv", True)][1] /
                                           max(1, prof[("spmv", True)][0]) * 1e-3) / 1e9,
        "setup_s": dict(setup, total=t_setup_total),
        "kernels": kernels,
        "instrumented_pass": {"ms_per_step": ms_prof / args.steps,
                              "kernel_time_fraction": total_prof / ms_prof,
                              "note": "per-kernel CUDA events on the launch stream; graph replay "
                                      "off during this pass"},
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(host_case_from_device(wl, prob, solver, b), solver,
                                           wl, iterations, threads=os.cpu_count() or 1)
    return out


def ncu_traffic(workload, kind):
    """dram__bytes_read+write of one launch of ``kind`` on ``workload``'s
    finest level, from an ncu --set full capture of that workload
    (profiles/ncu_traffic.json, keyed workload -> kernel); None when no
    capture of that workload/kernel exists."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        rec = json.load(f).get(workload) or {}
    v = rec.get(kind)
    return float(v) if v is not None else None


L2_BYTES = 126 * 2 ** 20

# BASELINE configs as benchmarked (both arms print the same ``config``);
# the deviations from the BASELINE text are explained in DESIGN.md
# ("Workloads").  finest_bytes: one finest-level SpMV + Vanka application
# (algorithmic), checked against the live figure in the device arm.
WORKLOADS = {
    "3d_large": dict(fine_mesh="128x32x32", levels=5, dofs=4343300, vanka_block="108x108",
                     dim=3, deform_taper=0.0, patches="fluid=one, solid=one",
                     sweep_bytes=23342906404),
    "3d_small": dict(fine_mesh="64x16x16", levels=4, dofs=561924, vanka_block="108x108",
                     dim=3, deform_taper=0.0, patches="fluid=one, solid=one",
                     sweep_bytes=2929533604),
    "2d_large": dict(fine_mesh="1024x256", levels=6, dofs=3153411, vanka_block="75x75",
                     dim=2, deform_taper=0.0625, patches="fluid=multi, solid=multi",
                     sweep_bytes=4624575692),
    "2d_small": dict(fine_mesh="256x64", levels=4, dofs=198531, vanka_block="75x75",
                     dim=2, deform_taper=0.0, patches="fluid=multi, solid=multi",
                     sweep_bytes=289250252),
    # the reference's 3D default blocking (newton.py:53-56) on a solid block
    # nested in the coarse grid (with the BASELINE box the
    # reference's own default-blocked MG-GMRES stalls)
    "3d_large_refblock": dict(fine_mesh="128x32x32", levels=5, dofs=4343300,
                              vanka_block="108x108 fluid + 500x500 solid", dim=3,
                              deform_taper=0.0, patches="fluid=one, solid=multi",
                              sweep_bytes=24533181732,
                              solid_box="[1,2]x[0,0.5]x[0,0.5] (corner block nested in the "
                                        "coarse grid, for 2x2x2-cell solid macro patches)"),
}


def workload_config(name, iterations, world):
    """``config`` of the JSON line, identical in both arms (same_config)."""
    w = WORKLOADS[name]
    d = w["dim"]
    box = "x".join(["[1,2]"] + ["[0.375,0.625]"] * (d - 1))
    return {"workload": name, "fine_mesh": w["fine_mesh"], "levels": w["levels"],
            "dofs": w["dofs"], "vanka_block": w["vanka_block"], "nu_pre": 2, "nu_post": 2,
            "omega": 0.8, "rel_tol": 1e-8, "gmres_iterations": iterations,
            "l2": (f"inputs larger than L2: a finest-level sweep streams operator + patch "
                   f"inverses of {w['sweep_bytes'] / 1e6:.0f} MB (> 126 MiB L2) from HBM "
                   f"every sweep; no flush"),
            "deviations": {"solid_box": w.get("solid_box", f"{box} (BASELINE [1,2]x[0.4,0.6]^"
                                                            f"{d - 1} snapped outward to the "
                                                            f"1/8 grid)"),
                           "lps_dt": 0.01, "deform_taper": w["deform_taper"],
                           "patches": w["patches"]},
            "parallelism": f"{world} independent replica(s)"}


# ------------------------------------------------------------------ CPU oracle baseline
def cpu_baseline(case, solver, wl, iterations, threads):
    """The oracle port (numpy/scipy restatement of the reference's gmres +
    MgSolver) on the same full hierarchy, host copies of the device-assembled
    operators and of the device's patch inverses (no CPU factorisation):
    a bounded sample of two complete Arnoldi steps of its gmres (V-cycle,
    operator product, classical Gram-Schmidt) plus one V-cycle, scaled to the
    solve's iteration count (iterations x step + final V-cycle)."""
    from oracle import linsolve_oracle as orc
    t_start = time.perf_counter()
    inverses = [None] + [[np.ascontiguousarray(solver.inverses(l, gi))
                          for gi in range(len(case.patches[l].groups))]
                         for l in range(1, len(case.matrices))]
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega, threads, inverses=inverses)
    t_prep = time.perf_counter() - t_start
    t0 = time.perf_counter()
    try:
        orc.gmres(mg.A[-1], case.b, mg, rel_tol=1e-300, max_iter=2)
    except orc.OracleSolverError:
        pass                      # two steps, then the final V-cycle; not converged
    t_two = time.perf_counter() - t0
    t0 = time.perf_counter()
    mg.dot(case.b)
    t_vc = time.perf_counter() - t0
    t_step = (t_two - t_vc) / 2
    t_solve = iterations * t_step + t_vc
    return {"value": 1.0 / t_solve, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"oracle port (numpy/scipy restatement of reference linsolve.py gmres + "
                       f"MgSolver) on the full {wl.name} hierarchy: 2 complete Arnoldi steps + "
                       f"final V-cycle ({t_two:.1f} s) and one V-cycle ({t_vc:.1f} s), scaled "
                       f"to {iterations} iterations; the measured complete solve of the "
                       f"unmodified reference is bench.py --impl reference"),
            "step_s": t_step, "vcycle_s": t_vc, "solve_s": t_solve, "prep_s": t_prep,
            "wall_s": time.perf_counter() - t_start}


# ----------------------------------------------------------------- reference arm (CPU)
def run_reference(args, rank, world):
    """The UNMODIFIED reference (baseline/_ref, pure Python) through its own
    API (baseline/ref_arm.py): problem, LinearStack.build_momentum, then
    complete gmres + MgSolver solves to 1e-8 on the box's host cores.  No
    import of the product package.  A step is one complete solve; the arm
    times as many as fit in --ref-budget-s (at least one) and reports the
    number actually timed."""
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "baseline"))
    import ref_arm
    if not ref_arm.available():
        return {"impl": "reference", "unavailable": "reference not installed in baseline/_ref"}
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    ref_arm.set_solve_threads(threads)
    stack, b, setup = ref_arm.build(args.workload, setup_threads=threads, log=log)
    t_setup = time.perf_counter() - t0
    log(f"[reference] setup {t_setup:.1f}s {setup}")
    solves, hist = [], None
    budget = args.ref_budget_s
    warm = 0
    tt = time.perf_counter()
    # A CPU solve has no warm-up effect that matters once it takes minutes
    # (no JIT, no lazy allocation in the timed code): a first solve longer
    # than a tenth of the budget is the first timed solve, otherwise the
    # requested warm-up solves run untimed first.
    while len(solves) < args.steps:
        ts = time.perf_counter()
        x, st = ref_arm.solve(stack, b)
        dt = time.perf_counter() - ts
        hist = st
        if not solves and warm < args.warmup and dt <= 0.1 * budget:
            warm += 1
            log(f"[reference] warm-up solve {dt:.1f}s, {st.iterations} iterations")
            tt = time.perf_counter()
            continue
        solves.append(dt)
        log(f"[reference] timed solve {dt:.1f}s, {st.iterations} iterations")
        if time.perf_counter() - tt + dt > budget:
            break
    t_timed = time.perf_counter() - tt
    parity = check_against_golden(args.workload, hist.iterations, hist.residuals,
                                  vector_checksums(x))
    value = len(solves) / t_timed
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": len(solves), "warmup": warm, "ms_per_step": 1e3 * t_timed / len(solves),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "impl": "reference",
            "data": f"synthetic (seeded sine-mode linearisation state and RHS, workload {args.workload})",
            "config": workload_config(args.workload, hist.iterations, world),
            "requested": {"steps": args.steps, "warmup": args.warmup,
                          "budget_s": budget},
            "parity": parity,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": (f"{len(solves)} complete solve(s) of the unmodified "
                                        f"reference (baseline/_ref: alefsi.linsolve.gmres + "
                                        f"MgSolver, rel_tol 1e-8) on {args.workload}, "
                                        f"{hist.iterations} GMRES iterations, BLAS + "
                                        f"_parallel.set_threads({threads}); setup (problem, "
                                        f"assembly, patch inverses, splu) {t_setup:.0f}s "
                                        f"untimed"),
                             "solve_s": solves, "setup_s": dict(setup, total=t_setup)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="3d_large")
    ap.add_argument("--sweeps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=900.0,
                    help="reference arm: wall-time budget of the timed solves (at least one)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        # rank 0 alone runs the CPU reference; no process group (a long CPU
        # run must not sit in a collective's timeout)
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group(backend="nccl")
    out = run_ours(args, rank, world)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
