#!/bin/bash
# round 2 (session 2): parity suite, default bench line, config-0/1 bench lines
OUT=${OUT:-s2a}
mkdir -p gpurun_out/$OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/$OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rs --durations=15 > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 600 python bench.py > gpurun_out/$OUT/bench_3d_large.json 2> gpurun_out/$OUT/bench_3d_large.err
for w in 2d_small 2d_large; do
  timeout 600 python bench.py --workload $w --steps 20 > gpurun_out/$OUT/bench_$w.json 2> gpurun_out/$OUT/bench_$w.err
done
echo done > gpurun_out/$OUT/done
