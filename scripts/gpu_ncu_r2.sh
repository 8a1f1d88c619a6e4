#!/bin/bash
# ncu evidence (round 2): launch list of config-0 solves; full capture of the
# 2D sliced-ELL SpMV (config 1 finest level) and of the 3D headline kernels.
OUT=${OUT:-r2n}
mkdir -p gpurun_out/$OUT
B0="python bench.py --workload 2d_small --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $B0 > gpurun_out/$OUT/plain_2d_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1200 --csv \
    --log-file gpurun_out/$OUT/launches_2d_small.csv $B0 > gpurun_out/$OUT/ncu_2d_small.log 2>&1
S1="python scripts/spmv_ab.py 2d_large --reps 3"
timeout 300 $S1 > gpurun_out/$OUT/plain_spmv.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv3_sell -s 2 -c 2 \
    -o gpurun_out/$OUT/spmv3_sell $S1 > gpurun_out/$OUT/ncu_spmv.log 2>&1
echo done > gpurun_out/$OUT/done
