#!/bin/bash
# round 2, final evidence: parity suite, bench lines of every workload on the
# final kernels (clock record per line), launch list of the default bench.
OUT=${OUT:-r2x}
mkdir -p gpurun_out/$OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/$OUT/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -rs --durations=10 > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 600 python bench.py > gpurun_out/$OUT/bench_3d_large.json 2> gpurun_out/$OUT/bench_3d_large.err
for w in 2d_small 2d_large 3d_small 3d_large_refblock; do
  timeout 900 python bench.py --workload $w --steps 20 > gpurun_out/$OUT/bench_$w.json 2> gpurun_out/$OUT/bench_$w.err
done
B3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/$OUT/launches_3d_large.csv $B3 > gpurun_out/$OUT/ncu_3d_large.log 2>&1
echo done > gpurun_out/$OUT/done
