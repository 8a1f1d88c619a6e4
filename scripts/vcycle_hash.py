"""SHA-256 of one device V-cycle and of a GMRES solve (A/B of bitwise-neutral
kernel variants on the GPU box).   python scripts/vcycle_hash.py [workload]"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1904_02401_b200 import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "3d_small"
    wl = W.CONFIGS[name]
    prob, mg, b, _ = W.build_device_solver(wl)
    z = mg.dot(b)
    x, st = mg.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    print(json.dumps({"workload": name,
                      "vcycle": hashlib.sha256(np.asarray(z).tobytes()).hexdigest()[:16],
                      "gmres_x": hashlib.sha256(np.asarray(x).tobytes()).hexdigest()[:16],
                      "iterations": st.iterations, "final": st.final_residual,
                      "elapsed": st.elapsed}), flush=True)


if __name__ == "__main__":
    main()
