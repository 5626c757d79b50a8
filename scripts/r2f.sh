#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
rm -f $OUT/zoo_*.ncu-rep
python scripts/kernel_zoo.py mass_k2 1 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:cellmat_tcs|geom_w_kernel" -c 2 -o $OUT/zoo_mass_tcs python scripts/kernel_zoo.py mass_k2 1 > $OUT/ncu_tcs.log 2>&1; echo "ncu rc=$?"
python scripts/zoo_summary.py r2f > /dev/null 2>&1; python - <<'PY'
import json
d = json.load(open("gpurun_out/r2f_zoo_summary.json"))
for e in d.get("mass_tcs", []):
    print("=====", e["kernel"][:70])
    for m, v in e.items():
        if m != "kernel": print("   ", m, v)
PY
ncu -i $OUT/zoo_mass_tcs.ncu-rep --page source --csv --kernel-name regex:cellmat_tcs > $OUT/tcs_source.csv 2>/dev/null; wc -l $OUT/tcs_source.csv
