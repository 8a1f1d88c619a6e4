"""Warm device assembly only (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1904_02401_b200 import workloads as W  # noqa: E402
wl = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "3d_small"]
prob, mg, b, _ = W.build_device_solver(wl)
U, Up = W.linearisation_state(wl, prob)
for l, lvl in enumerate(prob.levels):
    mg.asm_momentum(l, lvl, prob.mats, wl.dt, wl.theta, prob.restrict_state(U, l), prob.restrict_state(Up, l))
torch.cuda.synchronize()
