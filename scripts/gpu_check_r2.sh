#!/bin/bash
# GPU-box check used during round 2: parity suite, then measurements, then an
# ncu launch list of config-0 solves (host-stepped: ncu does not profile the
# kernels of a graph with conditional nodes).  Every step under a timeout.
OUT=${OUT:-r2}
mkdir -p gpurun_out/$OUT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 300 python scripts/spmv_ab.py 2d_large --reps 50 > gpurun_out/$OUT/spmv_2d_large.log 2>&1
for W in 3d_large 2d_small 2d_large 3d_small; do
  timeout 400 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline \
      > gpurun_out/$OUT/bench_$W.json 2> gpurun_out/$OUT/bench_$W.err
done
timeout 400 python scripts/fact_ab.py 3d_large 3d_small > gpurun_out/$OUT/fact.log 2>&1
B0="python bench.py --workload 2d_small --steps 2 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $B0 > gpurun_out/$OUT/plain_2d_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 1500 --csv \
    --log-file gpurun_out/$OUT/launches_2d_small.csv $B0 > gpurun_out/$OUT/ncu_2d_small.log 2>&1
echo done > gpurun_out/$OUT/done
