#!/bin/bash
# (1) ncu --set full of the finest-level 2D sliced-ELL SpMV (config 1) and of
#     the 3D headline SpMV / Vanka apply (config 3) on the current build;
# (2) the reference's own full solve of 3d_large_refblock on the box's host
#     cores (golden + setup digests), CPU only.
OUT=${OUT:-r2e}
mkdir -p gpurun_out/$OUT
S1="python scripts/spmv_ab.py 2d_large --reps 3"
timeout 300 $S1 > gpurun_out/$OUT/plain_spmv2d.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv3_sell -s 8 -c 1 \
    -o gpurun_out/$OUT/spmv3_sell_finest $S1 > gpurun_out/$OUT/ncu_spmv2d.log 2>&1
S3="python scripts/profile_kernels.py 3d_large --standalone"
timeout 600 $S3 > gpurun_out/$OUT/plain_3d.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:spmv4_kernel|vanka_apply_kernel" -s 4 -c 2 \
    -o gpurun_out/$OUT/headline_3d $S3 > gpurun_out/$OUT/ncu_3d.log 2>&1
mkdir -p gpurun_out/golden
timeout 2700 python tests/golden/make_golden_ref_arm.py 3d_large_refblock > gpurun_out/golden/refblock_log.txt 2>&1
echo rc=$? >> gpurun_out/golden/refblock_log.txt
echo done > gpurun_out/$OUT/done
