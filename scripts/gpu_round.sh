#!/bin/bash
# One GPU session: tests, bench, launch list, ncu full capture of the top kernels.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" ; tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json | head -c 3000; echo
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-assembly"
  $CMD > $OUT/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  $CMD > $OUT/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"cellmat_tc|geom_w" -s 6 -c 2 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
