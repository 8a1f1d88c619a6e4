"""Vanka + coarse factorisation timing on the GPU box (the A/B switches of
round 1 are gone from the library; DESIGN.md keeps their measurements).

    python scripts/fact_ab.py [workload ...]

Per workload: warm wall time of a full Vanka + coarse factorisation
(``mg.factorize()``, 5 repetitions) and SHA-256 of the GMRES solution and
residual history that follow it (bitwise comparison across variants).
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
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t = time.perf_counter()
            mg.factorize()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        sol, st = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=getattr(wl, "max_iter", 250))
        h = hashlib.sha256((sol.cpu().numpy() if hasattr(sol, "cpu") else np.asarray(sol)).tobytes()).hexdigest()[:16]
        hh = hashlib.sha256(np.asarray(st.residuals).tobytes()).hexdigest()[:16]
        print(json.dumps({"workload": name,
                          "factorize_s": ts, "its": st.iterations, "hash_x": h,
                          "hash_history": hh}), flush=True)
        del mg, prob
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
