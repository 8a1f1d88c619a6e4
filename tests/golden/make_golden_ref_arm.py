"""Golden fixtures for the BASELINE sizes the reference cannot run in the
build container (62 GB RAM): the UNMODIFIED reference installed in
``baseline/_ref`` is driven through ``baseline/ref_arm.py`` (the same
build/solve path as ``bench.py --impl reference``) on the GPU box's host
cores (196 GB RAM), e.g.

    gpurun -- python tests/golden/make_golden_ref_arm.py 3d_large 2d_large

and writes, per workload, into ``gpurun_out/golden/``:

* ``<w>.json``        the reference's full solve: iteration count, residual
                      history, solution checksums, setup / solve times;
* ``<w>_setup.json``  its index-structure digests and operator projections
                      on every level (same records as make_golden.py
                      --setup-only).

Nothing here imports ``paper_1904_02401_b200``.
"""

from __future__ import annotations

import json
import os
import resource
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline"))

import ref_arm  # noqa: E402
from golden_util import operator_checksums, sha, vector_checksums  # noqa: E402


def rss_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20


def run(name, out_dir, threads):
    t0 = time.perf_counter()
    ref_arm.set_solve_threads(threads)
    stack, b, tim = ref_arm.build(name, setup_threads=threads, log=print)
    t1 = time.perf_counter()
    print(name, f"setup {t1 - t0:.1f}s, peak RSS {rss_gb():.1f} GB", flush=True)
    x, st = ref_arm.solve(stack, b)
    t2 = time.perf_counter()
    print(name, f"solve {t2 - t1:.1f}s, {st.iterations} iterations", flush=True)
    solve = {"workload": name, "source": "reference (baseline/_ref via baseline/ref_arm.py)",
             "iterations": st.iterations, "residuals": [float(r) for r in st.residuals],
             "x_checksums": vector_checksums(x), "ndof": int(len(b)),
             "ref_setup_s": t1 - t0, "ref_setup_parts_s": tim, "ref_solve_s": t2 - t1,
             "threads": threads, "peak_rss_gb": rss_gb()}
    with open(os.path.join(out_dir, f"{name}.json"), "w") as f:
        json.dump(solve, f, indent=1)
    prob = stack.problem
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
    setup = {"workload": name, "source": "reference (setup, baseline/_ref via ref_arm.py)",
             "levels": levels, "ndof": int(len(b)), "ref_total_s": time.perf_counter() - t0}
    with open(os.path.join(out_dir, f"{name}_setup.json"), "w") as f:
        json.dump(setup, f, indent=1)
    print(name, "written", flush=True)


if __name__ == "__main__":
    out = os.path.join(ROOT, "gpurun_out", "golden")
    os.makedirs(out, exist_ok=True)
    threads = os.cpu_count() or 1
    for a in sys.argv[1:]:
        run(a, out, threads)
