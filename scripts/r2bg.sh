#!/bin/bash
set -u
OUT=gpurun_out
timeout 600 python scripts/kernel_zoo.py poisson_k2 1 > $OUT/zoo_pk2.plain 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:cellmat_tc2s" -c 1 -o $OUT/zoo_tc2s -f python scripts/kernel_zoo.py poisson_k2 1 > $OUT/zoo_tc2s.ncu.log 2>&1; echo "ncu rc=$?"
