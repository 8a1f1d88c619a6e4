#!/bin/bash
# GPU-box check used during round 2: parity suite, then measurements.
# Every step under its own timeout; outputs in gpurun_out/$OUT.
OUT=${OUT:-r2}
mkdir -p gpurun_out/$OUT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 300 python scripts/spmv_ab.py 2d_large --reps 50 > gpurun_out/$OUT/spmv_2d_large.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$OUT/bench_3d_large.json 2> gpurun_out/$OUT/bench_3d_large.err
timeout 300 python bench.py --workload 2d_small --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/$OUT/bench_2d_small.json 2> gpurun_out/$OUT/bench_2d_small.err
timeout 300 python bench.py --workload 2d_large --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$OUT/bench_2d_large.json 2> gpurun_out/$OUT/bench_2d_large.err
timeout 400 python scripts/fact_ab.py 3d_large 3d_small > gpurun_out/$OUT/fact.log 2>&1
echo done > gpurun_out/$OUT/done
