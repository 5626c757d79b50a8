#!/bin/bash
# Round-2a GPU session: GPU tests of the round-1 head, then `ncu --set full` of every kernel
# family DESIGN.md cites (mass K2, SIMT fp32/fp64, fused small-p, action, bounds, dofmap, CSR,
# scatter plan, deterministic / atomic / fused scatters), summarised on the box.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu.log
run() {  # kind regex count [skip]
  local kind=$1 re=$2 cnt=$3 skip=${4:-0}
  timeout 600 python scripts/kernel_zoo.py $kind 1 > $OUT/zoo_$kind.plain 2>&1 || { echo "$kind plain FAILED"; tail -3 $OUT/zoo_$kind.plain; return; }
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c $cnt \
    -o $OUT/zoo_$kind python scripts/kernel_zoo.py $kind 1 > $OUT/zoo_$kind.ncu.log 2>&1
  echo "$kind ncu rc=$?"
}
run mass_k2 "cellmat_tc2|geom_w_kernel" 2
run simt_f32 "cellmat_simt|geom_w_kernel" 2
run simt_f64 "cellmat_simt" 1
run fused_p1 "fused" 1
run action "action_kernel" 1
run bounds "bounds_kernel" 1
run asm_p2 ".*" 60
run asm_p3 "assemble|scatter|cellmat_tc2" 6
python scripts/zoo_summary.py r2a > $OUT/zoo_summary.txt 2>&1; echo "summary rc=$?"; head -c 4000 $OUT/zoo_summary.txt
mkdir -p /tmp/ncu_keep
for f in $OUT/zoo_*.ncu-rep; do
  sz=$(stat -c %s "$f")
  if [ "$sz" -gt 20000000 ]; then mv "$f" /tmp/ncu_keep/; fi
done
ls -la $OUT
