"""Device setup only (assembly + Vanka/coarse factorisation) for ncu launch lists."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_02401_b200 import workloads as W  # noqa: E402

wl = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "3d_large"]
prob, mg, b, t = W.build_device_solver(wl)
mg.factorize()
print(t, flush=True)
