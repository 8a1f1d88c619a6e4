"""Host-side setup profile of a workload (LevelData construction, patches,
transfers) — where the seconds before the first device kernel go."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1904_02401_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "3d_large"
wl = W.CONFIGS[name]
t = time.time()
prof = cProfile.Profile()
prof.enable()
prob = wl.problem()
prof.disable()
print(f"problem() {time.time() - t:.1f}s")
pstats.Stats(prof).sort_stats("cumulative").print_stats(30)
