#!/bin/bash
# round 2: config-4 device run (10 steps) + warm-cache launch list of config-0
# solves (host-stepped; --cache-control none keeps the L2-resident levels warm)
OUT=${OUT:-r2}
mkdir -p gpurun_out/$OUT
timeout 600 python scripts/timestep_run.py --out gpurun_out/$OUT/timestep_device.json \
    > gpurun_out/$OUT/timestep.log 2>&1
B0="python bench.py --workload 2d_small --steps 2 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $B0 > gpurun_out/$OUT/plain_2d_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    -s 2500 -c 1500 --csv --log-file gpurun_out/$OUT/launches_2d_small_warm.csv $B0 \
    > gpurun_out/$OUT/ncu_2d_small.log 2>&1
echo done > gpurun_out/$OUT/done
