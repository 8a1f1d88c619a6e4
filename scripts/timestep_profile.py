"""cProfile of the device time loop (config-4 family), for host-overhead work.

    python scripts/timestep_profile.py [--steps N] [--workload 3d_timestep]
"""
import argparse
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1904_02401_b200 import newton, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="3d_timestep")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    ts = W.TIMESTEPPING[args.workload]
    pr = cProfile.Profile()
    pr.enable()
    W.run_timestepping(ts, newton.LinearStack, n_steps=args.steps)
    pr.disable()
    st = pstats.Stats(pr, stream=open(args.out, "w") if args.out else sys.stdout)
    st.sort_stats("cumulative").print_stats(45)
    st.sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
