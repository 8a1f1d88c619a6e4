"""Per-level SpMV on the GPU box: hash and time every level's operator product.

    python scripts/spmv_ab.py [workload] [--reps N]

Prints one JSON line per level: SHA-256 of y = A x and of y = b - A x for a
seeded x (bitwise comparison across kernel variants) and the mean CUDA-event
time of N back-to-back products (algorithmic bytes / time as GB/s).
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
    name = next((a for a in sys.argv[1:] if not a.startswith("--")), "3d_large")
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 20
    wl = W.CONFIGS[name]
    t = time.time()
    prob, mg, b, _ = W.build_device_solver(wl)
    torch.cuda.synchronize()
    print(f"setup {time.time() - t:.1f}s", flush=True)
    for l, lvl in enumerate(prob.levels):
        p = lvl.pattern
        n = p.n_nodes * (wl.dim + 1)
        rng = np.random.default_rng(7 + l)
        x = torch.from_numpy(rng.standard_normal(n)).cuda()
        bb = torch.from_numpy(rng.standard_normal(n)).cuda()
        y0 = mg.spmv(l, x)
        y1 = mg.spmv(l, x, bb)
        torch.cuda.synchronize()
        h0 = hashlib.sha256(y0.cpu().numpy().tobytes()).hexdigest()[:16]
        h1 = hashlib.sha256(y1.cpu().numpy().tobytes()).hexdigest()[:16]
        nc = wl.dim + 1
        nnzb, npp = int(p.indptr[-1]), int(p.pp_indptr[-1]) if p.pp_indptr is not None else 0
        alg = nnzb * (nc * nc * 8 + 4) + (p.n_nodes + 1) * 8 + npp * 12 + 3 * n * 8
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            mg.spmv(l, x, bb, y1)
        e0.record()
        for _ in range(reps):
            mg.spmv(l, x, bb, y1)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"workload": name, "level": l, "nodes": p.n_nodes, "hash_Ax": h0, "hash_b_Ax": h1, "ms": ms,
                          "GBs": alg / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
