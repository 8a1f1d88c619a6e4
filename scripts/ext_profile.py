"""Per-kernel live timing (alefsi_mg_profile) of the harmonic-extension
MG-GMRES solve on the config-4 mesh, and its wall time per solve."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1904_02401_b200 import newton, workloads as W  # noqa: E402

ts = W.TIMESTEPPING[sys.argv[1] if len(sys.argv) > 1 else "3d_timestep"]
prob = ts.problem()
lin, nt, tl = ts.configs()
stack = newton.LinearStack(prob, lin)
stack._build_extension()
mg = stack.ext_mg.device if hasattr(stack.ext_mg, "device") else stack.ext_mg
n = prob.fine.n_nodes * prob.dim
rng = np.random.default_rng(0)
b = rng.standard_normal(n)
b[prob.levels[-1].ext_dirichlet.reshape(-1)] = 0.0
for _ in range(2):
    z, st = stack.solve_extension(b)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    z, st = stack.solve_extension(b)
torch.cuda.synchronize()
print("extension solve", st.iterations, "iterations", (time.perf_counter() - t) / 5 * 1e3, "ms")
dev = getattr(stack.ext_mg, "_dev", None) or getattr(stack.ext_mg, "dev", None) or mg
print(type(dev))
try:
    dev.profile(True)
    stack.solve_extension(b)
    pr = dev.profile_read()
    for k, v in sorted(pr.items(), key=lambda kv: -kv[1]["ms"] if isinstance(kv[1], dict) and "ms" in kv[1] else 0): print(k, v)
except Exception as e:
    print("profile unavailable:", e, [a for a in dir(stack.ext_mg) if not a.startswith("__")])
