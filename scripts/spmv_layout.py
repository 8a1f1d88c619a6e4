"""2D SpMV layout sweep on the GPU box: per level, time y = b - A x with the
CSR half-warp kernel (lanes 0) and sliced ELL with 1, 2, 4 lanes per row
(alefsi_mg_set_sell); prints one JSON line per (level, layout) with the
mean CUDA-event time, algorithmic GB/s and a hash of y (results of the
layouts differ only in the order a row's blocks are summed).

    python scripts/spmv_layout.py [workload ...] [--reps N]
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_02401_b200 import workloads as W  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("--") and not a.isdigit()] or ["2d_large"]
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 50
    for name in names:
        wl = W.CONFIGS[name]
        prob, mg, b, _ = W.build_device_solver(wl)
        for l, lvl in enumerate(prob.levels):
            p = lvl.pattern
            nc = wl.dim + 1
            n = p.n_nodes * nc
            rng = np.random.default_rng(7 + l)
            x = torch.from_numpy(rng.standard_normal(n)).cuda()
            bb = torch.from_numpy(rng.standard_normal(n)).cuda()
            y = torch.empty_like(x)
            alg = p.nnzb * (nc * nc * 8 + 4) + (p.n_nodes + 1) * 8 + p.nnz_pp * 12 + 3 * n * 8
            for lanes in (0, 1, 2, 4):
                mg.set_sell(l, lanes)
                for _ in range(3):
                    mg.spmv(l, x, bb, y)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    mg.spmv(l, x, bb, y)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                h = hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:12]
                print(json.dumps({"workload": name, "level": l, "nodes": p.n_nodes,
                                  "lanes": lanes, "ms": ms, "GBs": alg / ms / 1e6,
                                  "hash": h}), flush=True)
        del mg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
