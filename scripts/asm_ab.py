"""Warm device Jacobian assembly timing (all levels) + SHA-256 of the finest
level's assembled operator (bitwise comparison across kernel versions).

    python scripts/asm_ab.py [workload ...]
"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_02401_b200 import workloads as W  # noqa: E402


def main():
    for name in sys.argv[1:] or ["3d_small"]:
        wl = W.CONFIGS[name]
        prob, mg, b, _ = W.build_device_solver(wl)
        U, Up = W.linearisation_state(wl, prob)
        states = [(prob.restrict_state(U, l), prob.restrict_state(Up, l))
                  for l in range(len(prob.levels))]
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t = time.perf_counter()
            for l, lvl in enumerate(prob.levels):
                mg.asm_momentum(l, lvl, prob.mats, wl.dt, wl.theta, *states[l])
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        mg.factorize()
        sol, st = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=getattr(wl, "max_iter", 250))
        hh = hashlib.sha256(np.asarray(st.residuals).tobytes()).hexdigest()[:16]
        print(json.dumps({"workload": name, "assembly_ms": [round(1e3 * t, 2) for t in ts],
                          "its": st.iterations, "hash_history": hh}), flush=True)
        del mg, prob
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
