"""Generate the golden fixtures by running the UNMODIFIED reference
(/root/reference/pkg/src/alefsi) on the seeded workloads.

    python tests/golden/make_golden.py 2d_mini 2d_one 3d_tiny      # small, full detail
    python tests/golden/make_golden.py --solve-only 2d_small 3d_small
    python tests/golden/make_golden.py --setup-only 2d_small 2d_large 3d_small 3d_large
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py --tag=_t1 3d_timestep

The workload definition (box mesh arrays, seeded state and RHS) comes from
``paper_1904_02401_b200.workloads``; everything computed from it — node
numbering, patterns, patches, coloring, prolongation, assembled operators,
V-cycle, Vanka sweep and the GMRES residual history — is the reference's.
Exact integer structures are pinned by SHA-256 digests; floating-point
results by values (small cases) or by seeded projections (large cases).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import golden_util  # noqa: E402

HERE_OUT = [HERE]          # --out=DIR redirects the time-loop records
import refbridge as rb  # noqa: E402
from golden_util import sha, operator_checksums, vector_checksums  # noqa: E402
from paper_1904_02401_b200 import workloads as W  # noqa: E402


def run(name, solve_only=False):
    wl = W.CONFIGS[name]
    t0 = time.perf_counter()
    prob = rb.ref_problem(wl)
    # seeded state on the reference's own mesh (node coordinates)
    U, Up = W.linearisation_state(wl, prob)
    b = W.right_hand_side(wl, prob)
    stack = rb.ref_stack(wl, prob, U, Up)
    t1 = time.perf_counter()
    x, st = rb.ref_solve(wl, stack, b)
    t2 = time.perf_counter()
    out = {"workload": name, "iterations": st.iterations, "residuals": [float(r) for r in st.residuals],
           "x_checksums": vector_checksums(x), "ndof": int(len(b)),
           "ref_setup_s": t1 - t0, "ref_solve_s": t2 - t1}
    arrays = {}
    if not solve_only:
        mg = stack.mom_mg
        levels = []
        for l, lvl in enumerate(prob.levels):
            m = lvl.mesh
            rec = {"n_nodes": int(lvl.n_nodes),
                   "cell_nodes": sha(m.cell_nodes.astype(np.int64)),
                   "node_coords": sha(m.nodes.astype(np.float64)),
                   "node_class": sha(lvl.cls.node_class.astype(np.int8)),
                   "union_pattern": sha(lvl.pattern.indptr.astype(np.int64),
                                        lvl.pattern.indices.astype(np.int32)),
                   "momentum_dirichlet": sha(lvl.momentum_dirichlet.astype(np.uint8)),
                   "operator": operator_checksums(mg.levels[l].matrix)}
            if l > 0:
                sm = stack.mom_smoothers[l]
                rec["patches"] = [sha(g.astype(np.int64)) for g, _ in sm.patchset.groups]
                rec["patch_subdomains"] = [int(s) for _, s in sm.patchset.groups]
                rec["n_colors"] = int(sm.coloring.n_colors)
                rec["colors"] = sha(sm.coloring.color.astype(np.int64))
                P = stack.transfers[l].tocsr()
                P.sort_indices()
                rec["prolongation"] = sha(P.indptr.astype(np.int64), P.indices.astype(np.int32),
                                          P.data.astype(np.float64))
            levels.append(rec)
        out["levels"] = levels
        z = mg.dot(b)
        A = mg.levels[-1].matrix
        s1 = mg.levels[-1].smoother.sweep(A, np.zeros_like(b), b)
        s2 = mg.levels[-1].smoother.sweep(A, s1, b)
        out["vcycle_checksums"] = vector_checksums(z)
        out["sweep_checksums"] = vector_checksums(s2)
        if len(b) <= 20000:
            arrays = {"x": x, "vcycle": z, "sweep2": s2, "b": b}
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    if arrays:
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    print(name, "iterations", st.iterations, "setup %.1fs solve %.1fs" % (t1 - t0, t2 - t1))


def _blas_threads():
    try:
        import threadpoolctl
        return [i.get("num_threads") for i in threadpoolctl.threadpool_info()
                if i.get("user_api") == "blas"]
    except Exception:
        return None


def _block_projections(pattern, data, n_comp):
    """operator_checksums (u^T A v) of the reference's block operator,
    computed block-row-wise from its (nnzb, nc, nc) data without the
    CSR expansion (which does not fit in this container at config 3)."""
    n = pattern.n_nodes * n_comp
    us = golden_util.probe_vectors(n, 3, 1234)
    vs = golden_util.probe_vectors(n, 3, 4321)
    rows = np.asarray(pattern.rows)
    cols = np.asarray(pattern.cols)
    out = []
    for u, v in zip(us, vs):
        V = v.reshape(-1, n_comp)
        y = np.zeros((pattern.n_nodes, n_comp))
        step = 1 << 22
        for s in range(0, pattern.nnzb, step):
            e = min(s + step, pattern.nnzb)
            c = np.einsum("bij,bj->bi", data[s:e], V[cols[s:e]])
            for k in range(n_comp):
                y[:, k] += np.bincount(rows[s:e], weights=c[:, k], minlength=pattern.n_nodes)
        out.append(float(u @ y.reshape(-1)))
    return out


def run_setup(name, with_operator=True):
    """Setup only (no solve): the reference's index structures on every
    level (node numbering, union pattern, Dirichlet masks, patches,
    coloring, prolongation) and, optionally, projections of its assembled
    condensed Jacobian (reference model.py:297-381 through
    LinearStack.build_momentum's per-level data, newton.py:146-149)."""
    a = rb.ref()
    wl = W.CONFIGS[name]
    t0 = time.perf_counter()
    prob = rb.ref_problem(wl)
    U, Up = W.linearisation_state(wl, prob)
    fp, spt = wl.patch_strategies()
    cfg = a.newton.LinearConfig(fluid_patches=fp, solid_patches=spt, nu_pre=wl.nu_pre,
                                nu_post=wl.nu_post, omega=wl.omega, max_iter=wl.max_iter)
    stack = a.newton.LinearStack(prob, cfg)
    t1 = time.perf_counter()
    levels = []
    for l, lvl in enumerate(prob.levels):
        m = lvl.mesh
        rec = {"n_nodes": int(lvl.n_nodes),
               "cell_nodes": sha(m.cell_nodes.astype(np.int64)),
               "node_coords": sha(m.nodes.astype(np.float64)),
               "node_class": sha(lvl.cls.node_class.astype(np.int8)),
               "union_pattern": sha(lvl.pattern.indptr.astype(np.int64),
                                    lvl.pattern.indices.astype(np.int32)),
               "momentum_dirichlet": sha(lvl.momentum_dirichlet.astype(np.uint8))}
        if l > 0:
            sm = stack.mom_smoothers[l]
            rec["patches"] = [sha(g.astype(np.int64)) for g, _ in sm.patchset.groups]
            rec["patch_subdomains"] = [int(s) for _, s in sm.patchset.groups]
            rec["n_colors"] = int(sm.coloring.n_colors)
            rec["colors"] = sha(sm.coloring.color.astype(np.int64))
            P = stack.transfers[l].tocsr()
            P.sort_indices()
            rec["prolongation"] = sha(P.indptr.astype(np.int64), P.indices.astype(np.int32),
                                      P.data.astype(np.float64))
        if with_operator:
            data = a.model.momentum_jacobian_data(lvl, prob.mats, prob.flags, wl.dt, wl.theta,
                                                  prob.restrict_state(U, l),
                                                  prob.restrict_state(Up, l))
            rec["operator"] = _block_projections(lvl.pattern, data, wl.dim + 1)
            del data
        levels.append(rec)
        print(name, "level", l, "done %.1fs" % (time.perf_counter() - t0), flush=True)
    out = {"workload": name, "source": "reference (setup only)", "levels": levels,
           "ndof": int(prob.fine.n_nodes * (wl.dim + 1)),
           "ref_problem_stack_s": t1 - t0, "ref_total_s": time.perf_counter() - t0}
    with open(os.path.join(HERE, f"{name}_setup.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(name, "setup digests written %.1fs" % out["ref_total_s"])


def run_timestep(name, n_steps=None, tag="", threads=0):
    """The reference's run_time_loop on a TimeStepping workload (config 4
    family): per-step Newton/GMRES statistics and the final state.
    threads > 0: the reference's own patch-solve pool
    (alefsi._parallel.set_threads) and the bitwise-neutral batch split of
    numpy.einsum (baseline/ref_arm.threaded_einsum) — a different thread
    configuration of the same computation (run-to-run envelope)."""
    import contextlib
    ts = W.TIMESTEPPING[name]
    t0 = time.perf_counter()
    ctx = contextlib.nullcontext()
    if threads > 0:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(HERE)), "baseline"))
        import ref_arm
        rb.ref()._parallel.set_threads(threads)
        ctx = ref_arm.threaded_einsum(threads)
    def progress(records):
        # partial record after every time step (a multi-hour run survives an interruption)
        with open(os.path.join(HERE_OUT[0], f"{name}{tag}.partial.json"), "w") as f:
            json.dump({"workload": name, "records": records, "pool_threads": threads,
                       "blas_threads": _blas_threads(),
                       "ref_wall_s": time.perf_counter() - t0}, f, indent=1)

    with ctx:
        U, records = rb.ref_timestepping(ts, n_steps, on_record=progress)
    out = {"workload": name, "source": "reference run_time_loop", "n_steps": len(records),
           "records": records, "blas_threads": _blas_threads(), "pool_threads": threads,
           "U_checksums": vector_checksums(U.reshape(-1)), "ref_wall_s": time.perf_counter() - t0}
    with open(os.path.join(HERE_OUT[0], f"{name}{tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(name, [r["newton_steps"] for r in records], "%.1fs" % out["ref_wall_s"])


if __name__ == "__main__":
    args = sys.argv[1:]
    solve_only = "--solve-only" in args
    setup_only = "--setup-only" in args
    no_operator = "--no-operator" in args
    tag = next((a.split("=", 1)[1] for a in args if a.startswith("--tag=")), "")
    steps = next((int(a.split("=", 1)[1]) for a in args if a.startswith("--steps=")), None)
    threads = next((int(a.split("=", 1)[1]) for a in args if a.startswith("--threads=")), 0)
    out_dir = next((a.split("=", 1)[1] for a in args if a.startswith("--out=")), None)
    if out_dir:
        HERE_OUT[0] = out_dir
    for a in args:
        if a.startswith("--"):
            continue
        if a in W.TIMESTEPPING:
            run_timestep(a, steps, tag=tag, threads=threads)
        elif setup_only:
            run_setup(a, with_operator=not no_operator)
        else:
            run(a, solve_only)
