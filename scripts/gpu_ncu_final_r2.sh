#!/bin/bash
# ncu --set full of the final setup kernels at config 2's finest level:
# the 108x108 factorisation (slot-table gather) and the fluid assembly kernel
# (largest colour group).
OUT=${OUT:-r2x}
mkdir -p gpurun_out/$OUT
P2="python scripts/profile_setup_kernels.py 3d_small"
timeout 300 $P2 > gpurun_out/$OUT/plain_setup_3d_small.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vanka_factorize_pw -s 3 -c 1 \
    -o gpurun_out/$OUT/fact108 $P2 > gpurun_out/$OUT/ncu_fact108.log 2>&1
PA="python scripts/profile_asm.py 3d_small"
timeout 300 $PA > gpurun_out/$OUT/plain_asm_3d_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:assemble_cells --csv \
    --log-file gpurun_out/$OUT/asm_launches.csv $PA > gpurun_out/$OUT/ncu_asm_list.log 2>&1
echo done > gpurun_out/$OUT/done
