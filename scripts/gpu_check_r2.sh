#!/bin/bash
# GPU-box check used during round 2: parity suite, 2D SpMV layout sweep, the
# driver's default bench line (with cpu_baseline), per-config bench lines,
# factorisation timings.  Every step under its own timeout.
OUT=${OUT:-r2}
mkdir -p gpurun_out/$OUT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -rs > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 400 python scripts/spmv_layout.py 2d_large 2d_small --reps 50 > gpurun_out/$OUT/spmv_layout.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/$OUT/bench_default.json 2> gpurun_out/$OUT/bench_default.err
timeout 300 python bench.py --workload 2d_small --steps 200 --warmup 5 --no-cpu-baseline \
    > gpurun_out/$OUT/bench_2d_small.json 2> gpurun_out/$OUT/bench_2d_small.err
for W in 2d_large 3d_small 3d_large_refblock; do
  timeout 400 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline \
      > gpurun_out/$OUT/bench_$W.json 2> gpurun_out/$OUT/bench_$W.err
done
timeout 500 python scripts/fact_ab.py 3d_large 3d_small 3d_large_refblock > gpurun_out/$OUT/fact.log 2>&1
echo done > gpurun_out/$OUT/done
