#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
rm -f $OUT/*.ncu-rep
python scripts/kernel_zoo.py poisson_k2 1 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:geom_w_kernel" -c 1 -o $OUT/k1_poisson python scripts/kernel_zoo.py poisson_k2 1 > $OUT/ncu_k1.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/k1_poisson.ncu-rep --page source --csv > $OUT/k1_source.csv 2>/dev/null; wc -l $OUT/k1_source.csv
ncu -i $OUT/k1_poisson.ncu-rep --page raw --csv > $OUT/k1_raw.csv 2>/dev/null; wc -l $OUT/k1_raw.csv
