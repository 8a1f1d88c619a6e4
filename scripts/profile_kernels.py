"""Workload driver for ncu captures (run under gpurun).

    python scripts/profile_kernels.py [workload] [--standalone]

Default: one MG-GMRES solve of the workload (for the per-launch time list).
--standalone: only finest-level kernels — 3 Vanka sweeps then 3 SpMVs —
for `ncu --set full` captures of the two dominant kernels.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1904_02401_b200 import workloads as W  # noqa: E402


def main():
    name = next((a for a in sys.argv[1:] if not a.startswith("--")), "3d_large")
    standalone = "--standalone" in sys.argv
    wl = W.CONFIGS[name]
    t = time.time()
    prob, solver, bh, _ = W.build_device_solver(wl)      # the bench.py path
    b = torch.from_numpy(bh).cuda()
    torch.cuda.synchronize()
    print(f"setup {time.time() - t:.1f}s", flush=True)
    L = solver.n_levels - 1
    if standalone:
        x = torch.zeros_like(b)
        for _ in range(3):
            solver.sweep(L, x, b)
        y = torch.empty_like(b)
        for _ in range(3):
            solver.spmv(L, x, None, y)
    else:
        x, st = solver.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
        print("iterations", st.iterations, flush=True)
    torch.cuda.synchronize()
    print("done", flush=True)


if __name__ == "__main__":
    main()
