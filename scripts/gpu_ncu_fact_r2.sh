#!/bin/bash
# ncu evidence for the second-form patch factorisation kernels (round 2,
# session 3): launch list of config-3 setup + one --set full capture of the
# 108x108 kernel (config 2 finest level) and of the 75x75 kernel (config 0).
OUT=${OUT:-r2h}
mkdir -p gpurun_out/$OUT
P3="python scripts/profile_setup_kernels.py 3d_large"
timeout 300 $P3 > gpurun_out/$OUT/plain_3d_large.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/$OUT/launches_setup_3d_large.csv $P3 > gpurun_out/$OUT/ncu_launches.log 2>&1
P2="python scripts/profile_setup_kernels.py 3d_small"
timeout 300 $P2 > gpurun_out/$OUT/plain_3d_small.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vanka_factorize_pw -s 3 -c 1 \
    -o gpurun_out/$OUT/fact108 $P2 > gpurun_out/$OUT/ncu_fact108.log 2>&1
P0="python scripts/profile_setup_kernels.py 2d_large"
timeout 300 $P0 > gpurun_out/$OUT/plain_2d_large.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vanka_factorize_pw -s 5 -c 1 \
    -o gpurun_out/$OUT/fact75 $P0 > gpurun_out/$OUT/ncu_fact75.log 2>&1
echo done > gpurun_out/$OUT/done
