"""Development A/B of the 108x108 patch factorisation kernels on the GPU box.

    python scripts/fact_variants.py [workload ...]

Per workload and variant (0 = column-strided kernel, 12 / 9 = panel-of-warp
kernel with that many warps): warm wall time of ``mg.factorize()`` (5
repetitions), max relative difference of the finest level's stored inverses
against variant 0, and the GMRES iteration count / history difference of the
solve that follows.
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_02401_b200 import _lib, workloads as W  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["3d_small"]
    variants = [int(a[11:]) for a in sys.argv if a.startswith("--variants=")] or [0, 6, 106, 104]
    lib = _lib.load()
    setv = lib.alefsi_dev_set_fact_variant
    setv.argtypes = [ctypes.c_int]
    setv.restype = None
    for name in names:
        wl = W.CONFIGS[name]
        prob, mg, b, _ = W.build_device_solver(wl)
        ref_inv, ref_hist = None, None
        top = len(prob.levels) - 1
        for v in variants:
            setv(v)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                t = time.perf_counter()
                mg.factorize()
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t)
            sol, st = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=getattr(wl, "max_iter", 250))
            hist = np.asarray(st.residuals)
            inv = mg.inverses(top, 0)[:2048].copy()
            rec = {"workload": name, "variant": v, "factorize_ms": [round(1e3 * t, 2) for t in ts],
                   "its": st.iterations}
            if ref_inv is None:
                ref_inv, ref_hist = inv, hist
            else:
                scale = np.abs(ref_inv).max(axis=(1, 2), keepdims=True)
                rec["inv_max_rel_diff"] = float((np.abs(inv - ref_inv) / scale).max())
                rec["hist_max_rel_diff"] = (float(np.max(np.abs(hist - ref_hist) / ref_hist))
                                            if len(hist) == len(ref_hist) else None)
            print(json.dumps(rec), flush=True)
        setv(0)
        del mg, prob
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
