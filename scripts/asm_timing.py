"""Per-piece wall times of LinearStack.build_momentum on the config-4 mesh
(host outflow blocks, C-ABI assembly call per level, factorisation)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_02401_b200 import _lib, fem, model, newton, workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "3d_timestep"
    ts = W.TIMESTEPPING[name]
    prob = ts.problem()
    lin, nt, tl = ts.configs()
    stack = newton.LinearStack(prob, lin)
    U = prob.zero_state()
    prob.impose_boundary_values(U, 0.01)
    rng = np.random.default_rng(0)
    U[:, 1:] += 1e-3 * rng.standard_normal(U[:, 1:].shape)
    Up = prob.zero_state()
    k, theta = ts.base.dt, 0.5 + 2 * ts.base.dt
    t = time.perf_counter()
    stack.build_momentum(U, Up, k, theta)
    torch.cuda.synchronize()
    print(f"first build_momentum {time.perf_counter() - t:.3f}s")
    mg = stack.mom_mg
    for rep in range(3):
        tt = {}
        for l, lvl in enumerate(prob.levels):
            t = time.perf_counter()
            Ul, Upl = prob.restrict_state(U, l), prob.restrict_state(Up, l)
            tt[f"restrict{l}"] = time.perf_counter() - t
            if lvl.outflow is not None:
                t = time.perf_counter()
                with fem.single_blas():
                    model._outflow_blocks(lvl.outflow, Ul, prob.mats, k, theta, lvl.dim)
                tt[f"outflow{l}"] = time.perf_counter() - t
            t = time.perf_counter()
            mg.asm_momentum(l, lvl, prob.mats, k, theta, Ul, Upl)
            tt[f"asm{l}"] = time.perf_counter() - t
        t = time.perf_counter()
        mg.factorize()
        tt["factorize"] = time.perf_counter() - t
        t = time.perf_counter()
        stack.build_momentum(U, Up, k, theta)
        tt["build_momentum"] = time.perf_counter() - t
        print({a: round(b * 1e3, 2) for a, b in tt.items()})


if __name__ == "__main__":
    main()
