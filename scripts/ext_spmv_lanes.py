"""Sliced-ELL lanes-per-row sweep of the harmonic-extension operator's SpMV
(nc = 3, 3D cell stencil: 64 blocks per row) on the config-4 mesh."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1904_02401_b200 import newton, workloads as W  # noqa: E402

ts = W.TIMESTEPPING[sys.argv[1] if len(sys.argv) > 1 else "3d_timestep"]
prob = ts.problem()
lin, nt, tl = ts.configs()
stack = newton.LinearStack(prob, lin)
stack._build_extension()
mg = stack.ext_mg
top = len(prob.levels) - 1
for level in (top, top - 1):
    n = prob.levels[level].n_nodes * prob.dim
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ref = None
    for lanes in (0, 1, 2, 4):
        try:
            mg.set_sell(level, lanes)
        except Exception as e:
            print(level, lanes, "unavailable:", e)
            continue
        for _ in range(3):
            mg.spmv(level, x, None, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            mg.spmv(level, x, None, y)
        e1.record()
        torch.cuda.synchronize()
        yy = y.clone()
        if ref is None:
            ref = yy
        print("level", level, "nodes", prob.levels[level].n_nodes, "lanes", lanes,
              "%.1f us" % (e0.elapsed_time(e1) / 50 * 1e3),
              "max diff vs first", float((yy - ref).abs().max()), flush=True)
