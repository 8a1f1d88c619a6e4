"""Vanka apply form sweep on the GPU box: per level, the apply time of the
unsplit and the column-split kernel (alefsi_mg_set_apply_split), from the
library's per-kernel CUDA events over N sweeps, and the GMRES solve time
with each form on the finest level.

    python scripts/apply_layout.py [workload ...] [--reps N]
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
    names = [a for a in sys.argv[1:] if not a.startswith("--") and not a.isdigit()] or ["2d_small"]
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 50
    for name in names:
        wl = W.CONFIGS[name]
        prob, mg, b, _ = W.build_device_solver(wl, use_graph=True)
        mg.reserve(wl.max_iter)
        bd = torch.from_numpy(b).cuda()
        for l in range(1, len(prob.levels)):
            n = prob.levels[l].n_nodes * (wl.dim + 1)
            bl = torch.from_numpy(np.random.default_rng(l).standard_normal(n)).cuda()
            for split in (0, 1):
                mg.set_apply_split(l, split)
                x = torch.zeros_like(bl)
                mg.sweep(l, x, bl)
                mg.profile(True)
                mg.profile_read(reset=True)
                for _ in range(reps):
                    mg.sweep(l, x, bl)
                torch.cuda.synchronize()
                prof = mg.profile_read(reset=True)
                mg.profile(False)
                finest = l == len(prob.levels) - 1
                cnt, ms = prof[("vanka_apply", finest)]
                print(json.dumps({"workload": name, "level": l, "split": split,
                                  "apply_us": 1e3 * ms / max(cnt, 1)}), flush=True)
            mg.set_apply_split(l, -1)
        L = len(prob.levels) - 1
        for split in (-1, 0, 1):
            mg.set_apply_split(L, split)
            for _ in range(3):
                mg.gmres(bd, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                x, st = mg.gmres(bd, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"workload": name, "finest_split": split, "iterations": st.iterations,
                              "solve_ms": e0.elapsed_time(e1) / reps}), flush=True)
        mg.set_apply_split(L, -1)
        del mg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
