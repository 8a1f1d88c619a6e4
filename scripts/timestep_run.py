"""BASELINE config 4: 10 implicit time steps on the config-2 mesh.

    python scripts/timestep_run.py [--oracle] [--steps N] [--workload 3d_timestep] [--out F]

Device run (default): momentum and harmonic-extension MG-GMRES solves on the
GPU through newton.LinearStack.  --oracle: the same loop with the CPU oracle's
linear stack (test infrastructure; used to produce the comparison record).
Prints one JSON record per step and a summary line.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1904_02401_b200 import newton, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="3d_timestep")
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    ts = W.TIMESTEPPING[args.workload]
    if args.oracle:
        from oracle import linsolve_oracle as orc
        factory = lambda p, c: orc.OracleLinearStack(p, c, threads=args.threads)  # noqa: E731
    else:
        factory = newton.LinearStack
    t0 = time.perf_counter()

    def on_step(rec, U):
        print(json.dumps(rec), flush=True)
    from golden_like import vector_checksums
    U, recs = W.run_timestepping(ts, factory, on_step=on_step, n_steps=args.steps)
    out = {"workload": args.workload, "impl": "oracle" if args.oracle else "device",
           "n_steps": len(recs), "records": recs, "wall_s": time.perf_counter() - t0,
           "U_checksums": vector_checksums(U.reshape(-1))}
    print(json.dumps({k: v for k, v in out.items() if k != "records"}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tests"))
    import golden_util as golden_like  # noqa: F401
    sys.modules["golden_like"] = golden_like
    main()
