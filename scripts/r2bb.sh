#!/bin/bash
set -u
OUT=gpurun_out
timeout 600 python scripts/kernel_zoo.py action 1 > $OUT/zoo_action.plain 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --section SourceCounters --section InstructionStats --section WarpStateStats --import-source on --clock-control none -k regex:action_kernel -c 1 -o $OUT/action_src -f python scripts/kernel_zoo.py action 1 > $OUT/action_src.log 2>&1; echo "ncu rc=$?"; ls -la $OUT/action_src.ncu-rep
