#!/bin/bash
# ncu captures for profiles/r1g: launch list of the bench step, full set of K1/K2 and of the
# action kernel (config 1, mixed). Reports stay small enough to travel back (< 64 MiB).
set -u
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-assembly --no-modes --no-action --no-hex"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"cellmat_tc|geom_w" -s 6 -c 2 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/action_prof.py mixed > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:action_kernel -s 3 -c 1 -o $OUT/prof_action python scripts/action_prof.py mixed > $OUT/ncu_action.log 2>&1; echo "ncu action rc=$?"

# summarise on the box (the full reports exceed gpurun's 64 MiB return limit)
NCU_SUMMARY_DIR=$OUT python scripts/ncu_summary.py r1g "$CMD" > /dev/null && echo "summary ok"
ncu -i $OUT/prof_action.ncu-rep --page details --csv > $OUT/action_details.csv 2>/dev/null
mkdir -p /tmp/ncu_keep && mv $OUT/prof.ncu-rep /tmp/ncu_keep/

ls -la $OUT
