#!/bin/bash
# The reference's own complete 10-step config-4 run with a 16-thread patch
# pool + einsum split on the GPU box's host cores (second thread configuration
# of the same computation; partial record after every step).
mkdir -p gpurun_out/golden
timeout 10200 python tests/golden/make_golden.py --threads=16 --tag=_t16 \
    --out=gpurun_out/golden 3d_timestep > gpurun_out/golden/ts10_log.txt 2>&1
echo rc=$? >> gpurun_out/golden/ts10_log.txt
