#!/bin/bash
# round 2: parity suite, Vanka apply form sweep, and the reference's own
# first two config-4 time steps with a different thread configuration
# (16-thread patch pool + BLAS + einsum split) on the box's host cores
OUT=${OUT:-r2}
mkdir -p gpurun_out/$OUT gpurun_out/golden
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -rs > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 600 python scripts/apply_layout.py 2d_small 2d_large --reps 30 > gpurun_out/$OUT/apply_layout.log 2>&1
timeout 2400 python tests/golden/make_golden.py --threads=16 --steps=2 --tag=_2steps_t16 \
    --out=gpurun_out/golden 3d_timestep > gpurun_out/golden/ts2_log.txt 2>&1
echo rc=$? >> gpurun_out/golden/ts2_log.txt
echo done > gpurun_out/$OUT/done
