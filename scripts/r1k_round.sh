#!/bin/bash
# Round-1h GPU session: GPU tests, the default bench line (hex table with the accessor K1-box),
# the launch list, and ncu --set full of K1-box (Q2 Poisson hexes) beside K1/K2 of the headline.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-assembly --no-modes --no-action --no-hex"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"cellmat_tc|geom_w_kernel" -s 6 -c 2 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
HCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-assembly --no-modes --no-action"
ncu --set full --clock-control none --import-source on -k regex:geom_w_box -s 60 -c 1 -o $OUT/prof_box $HCMD > $OUT/ncu_box.log 2>&1; echo "ncu box rc=$?"
NCU_SUMMARY_DIR=$OUT python scripts/ncu_summary.py r1k "$CMD" > /dev/null && echo "summary ok"
python - <<'PY'
import sys; sys.path.insert(0, "scripts")
import json, ncu_summary as s
print(json.dumps(s.full("gpurun_out/prof_box.ncu-rep"), indent=1))
PY
ncu -i $OUT/prof_box.ncu-rep --page source --csv > $OUT/box_source.csv 2>/dev/null
mkdir -p /tmp/ncu_keep && mv $OUT/prof.ncu-rep $OUT/prof_box.ncu-rep /tmp/ncu_keep/ 2>/dev/null
ls -la $OUT
