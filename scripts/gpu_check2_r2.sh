#!/bin/bash
# round 2: parity suite, benches, and an ncu launch list of the refblock
# factorisation (500x500 macro-patch kernels)
OUT=${OUT:-r2}
mkdir -p gpurun_out/$OUT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -rs > gpurun_out/$OUT/pytest.log 2>&1
echo rc=$? >> gpurun_out/$OUT/pytest.log
timeout 300 python bench.py --workload 2d_small --steps 200 --warmup 5 --no-cpu-baseline \
    > gpurun_out/$OUT/bench_2d_small.json 2> gpurun_out/$OUT/bench_2d_small.err
for W in 2d_large 3d_large_refblock; do
  timeout 400 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline \
      > gpurun_out/$OUT/bench_$W.json 2> gpurun_out/$OUT/bench_$W.err
done
F="python scripts/fact_ab.py 3d_large_refblock"
timeout 400 $F > gpurun_out/$OUT/plain_fact.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/$OUT/launches_fact_refblock.csv $F > gpurun_out/$OUT/ncu_fact.log 2>&1
echo done > gpurun_out/$OUT/done
