#!/bin/bash
set -u
OUT=gpurun_out
timeout 600 python scripts/pull_prof.py 3 > $OUT/pull_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:assemble_pull -c 1 -s 1 -o $OUT/pull_p3 -f python scripts/pull_prof.py 3 > $OUT/pull_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $OUT/pull_ncu.log
