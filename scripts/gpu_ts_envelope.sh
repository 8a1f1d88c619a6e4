#!/bin/bash
# The reference's own first two config-4 time steps with a different thread
# configuration (16-thread patch pool + einsum split, BLAS threads as the box
# sets them) on the GPU box's host cores: the run-to-run envelope of the
# stagnating Newton solve at t = 0.02.
mkdir -p gpurun_out/golden
timeout 3300 python tests/golden/make_golden.py --threads=16 --steps=2 --tag=_2steps_t16 \
    --out=gpurun_out/golden 3d_timestep > gpurun_out/golden/ts2_log.txt 2>&1
echo rc=$? >> gpurun_out/golden/ts2_log.txt
