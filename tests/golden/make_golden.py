"""Generate the golden fixtures by running the UNMODIFIED reference
(/root/reference/pkg/src/alefsi) on the seeded workloads.

    python tests/golden/make_golden.py 2d_mini 2d_one 3d_tiny      # small, full detail
    python tests/golden/make_golden.py --solve-only 2d_small 3d_small

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


def run_timestep(name, n_steps=None):
    """The reference's run_time_loop on a TimeStepping workload (config 4
    family): per-step Newton/GMRES statistics and the final state."""
    ts = W.TIMESTEPPING[name]
    t0 = time.perf_counter()
    U, records = rb.ref_timestepping(ts, n_steps)
    out = {"workload": name, "n_steps": len(records), "records": records,
           "U_checksums": vector_checksums(U.reshape(-1)), "ref_wall_s": time.perf_counter() - t0}
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(name, [r["newton_steps"] for r in records], "%.1fs" % out["ref_wall_s"])


if __name__ == "__main__":
    args = sys.argv[1:]
    solve_only = "--solve-only" in args
    for a in args:
        if a.startswith("--"):
            continue
        if a in W.TIMESTEPPING:
            run_timestep(a)
        else:
            run(a, solve_only)
