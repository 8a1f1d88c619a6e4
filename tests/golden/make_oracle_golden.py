"""Full-size golden records from the CPU oracle (for workloads too large for
the unmodified reference in this container, e.g. the 4.3M-dof headline).

    python tests/golden/make_oracle_golden.py 3d_large [threads]

The oracle itself is pinned to the reference by the fixtures of
make_golden.py (iteration counts and residual histories to <1e-12 on every
case the reference can run here, including configs 0 and 2 at full size).
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from golden_util import vector_checksums  # noqa: E402
from oracle import linsolve_oracle as orc  # noqa: E402
from paper_1904_02401_b200 import workloads as W  # noqa: E402


def main():
    name = sys.argv[1]
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    wl = W.CONFIGS[name]
    t0 = time.perf_counter()
    case = W.build_case(wl, with_coloring=False)
    t1 = time.perf_counter()
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega, threads)
    t2 = time.perf_counter()
    x, st = orc.gmres(mg.A[-1], case.b, mg, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    t3 = time.perf_counter()
    out = {"workload": name, "source": "oracle", "iterations": st.iterations,
           "residuals": [float(r) for r in st.residuals], "x_checksums": vector_checksums(x),
           "ndof": int(len(case.b)), "threads": threads,
           "host_case_s": t1 - t0, "oracle_setup_s": t2 - t1, "oracle_solve_s": t3 - t2}
    with open(os.path.join(HERE, f"{name}_oracle.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(name, st.iterations, f"case {t1 - t0:.0f}s setup {t2 - t1:.0f}s solve {t3 - t2:.0f}s")


if __name__ == "__main__":
    main()
