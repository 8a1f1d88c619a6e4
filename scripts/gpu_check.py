"""Quick device-vs-oracle check used during development (GPU box)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_02401_b200 import workloads as W, device
from oracle import linsolve_oracle as orc

for name in sys.argv[1:]:
    wl = W.CONFIGS[name]
    t = time.time(); case = W.build_case(wl); tc = time.time() - t
    t = time.time(); solver = device.DeviceMgSolver.from_case(case, wl); tf = time.time() - t
    mg = orc.MgOracle(case, wl.nu_pre, wl.nu_post, wl.omega)
    b = case.b
    z = solver.dot(b); zo = mg.dot(b)
    print(name, "case %.2fs setup+factorize %.2fs" % (tc, tf), "vcycle rel diff", np.linalg.norm(z - zo) / np.linalg.norm(zo), flush=True)
    x, st = solver.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    xo, so = orc.gmres(mg.A[-1], b, mg, rel_tol=wl.rel_tol, max_iter=wl.max_iter)
    r1, r2 = np.array(st.residuals), np.array(so.residuals)
    n = min(len(r1), len(r2))
    print(name, "its", st.iterations, so.iterations, "hist maxrel", np.max(np.abs(r1[:n] - r2[:n]) / r2[:n]),
          "x rel", np.linalg.norm(x - xo) / np.linalg.norm(xo), "gpu solve %.4fs" % st.elapsed, flush=True)
    ts = []
    for _ in range(3):
        x, st = solver.gmres(b, rel_tol=wl.rel_tol, max_iter=wl.max_iter); ts.append(st.elapsed)
    print(name, "gmres e2e times", ts, "launches", solver.kernel_launches(), flush=True)
