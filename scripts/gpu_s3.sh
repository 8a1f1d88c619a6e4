#!/bin/bash
# round 2 (session 3): parity suite, factorisation timing, default bench line
OUT=${OUT:-s3}
mkdir -p gpurun_out/$OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/$OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rs --durations=15 > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 300 python scripts/fact_ab.py 2d_small 2d_large 3d_small 3d_large > gpurun_out/$OUT/fact.log 2>&1
timeout 600 python bench.py > gpurun_out/$OUT/bench_3d_large.json 2> gpurun_out/$OUT/bench_3d_large.err
echo done > gpurun_out/$OUT/done
