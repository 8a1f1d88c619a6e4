"""Coarse-level inverse check on the GPU box.

    python scripts/coarse_ab.py [workload]

Prints the warm time of a full Vanka + coarse factorisation, the coarse solve
of a seeded vector (norm, a few entries, and its relative residual against
the assembled coarse operator) and the GMRES history of the workload solve.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_02401_b200 import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "3d_small"
    wl = W.CONFIGS[name]
    prob, mg, b, _ = W.build_device_solver(wl)
    n0 = prob.levels[0].pattern.n_nodes * (wl.dim + 1)
    rhs = np.random.default_rng(3).standard_normal(n0)
    x = torch.from_numpy(rhs).cuda()
    y = torch.empty_like(x)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        mg.factorize()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    mg.coarse_solve(x, y)
    r = mg.spmv(0, y, x)          # x - A0 y
    torch.cuda.synchronize()
    sol, st = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    print(json.dumps({"workload": name,
                      "coarse_dofs": n0, "factorize_s": ts,
                      "coarse_rel_residual": float(torch.linalg.norm(r) / torch.linalg.norm(x)),
                      "y_head": y[:4].cpu().tolist(), "its": st.iterations,
                      "history": st.residuals}), flush=True)


if __name__ == "__main__":
    main()
