#!/bin/bash
# Round-1d GPU session: full GPU tests, default bench, launch list, ncu full captures of
# K1/K2 (headline) and the action kernel.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; head -c 600 $OUT/bench.json; echo
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-assembly --no-modes"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
$CMD > $OUT/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cellmat_tc|geom_w" -s 6 -c 2 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/action_prof.py mixed > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:action_kernel -s 1 -c 3 -o $OUT/prof_action python scripts/action_prof.py mixed > $OUT/ncu_action.log 2>&1; echo "ncu action rc=$?"
