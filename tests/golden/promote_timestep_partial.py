"""Promote the per-step partial record of a running / interrupted reference
time loop (make_golden.py writes <name><tag>.partial.json after every step)
to a golden fixture holding the completed steps:

    python tests/golden/promote_timestep_partial.py build/ts/3d_timestep_refA.partial.json \
        tests/golden/3d_timestep.json
"""
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
with open(src) as f:
    d = json.load(f)
out = {"workload": d["workload"], "source": "reference run_time_loop (stock thread configuration; "
       "record of the completed steps of a run still in progress / interrupted)",
       "n_steps": len(d["records"]), "records": d["records"], "blas_threads": d.get("blas_threads"),
       "pool_threads": d.get("pool_threads", 0), "ref_wall_s": d.get("ref_wall_s")}
with open(dst, "w") as f:
    json.dump(out, f, indent=1)
print(dst, out["n_steps"], "steps", [r["newton_steps"] for r in out["records"]])
