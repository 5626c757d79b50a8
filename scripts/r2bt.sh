#!/bin/bash
# Round-2 final GPU session: full GPU tests, default bench line, reference arm, config-2 sweep,
# launch list, ncu --set full of every kernel family (zoo).
set -u
OUT=gpurun_out
mkdir -p $OUT
rm -f $OUT/*.ncu-rep
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -2 $OUT/bench.err; head -c 800 $OUT/bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; head -c 600 $OUT/bench_ref.json; echo
timeout 1500 python bench.py --steps 5 --sweep --robustness --no-assembly --no-action --no-hex --no-modes --no-cpu-baseline > $OUT/bench_sweep.json 2> $OUT/bench_sweep.err; echo "sweep rc=$?"; tail -2 $OUT/bench_sweep.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-assembly --no-modes --no-action --no-hex"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
run() {  # kind regex count
  local kind=$1 re=$2 cnt=$3
  timeout 600 python scripts/kernel_zoo.py $kind 1 > $OUT/zoo_$kind.plain 2>&1 || { echo "$kind plain FAILED"; tail -3 $OUT/zoo_$kind.plain; return; }
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$re" -c $cnt \
    -o $OUT/zoo_$kind python scripts/kernel_zoo.py $kind 1 > $OUT/zoo_$kind.ncu.log 2>&1
  echo "$kind ncu rc=$?"
}
run poisson_k2 "cellmat_tc2|geom_w_kernel" 2
run mass_k2 "cellmat_tcs|geom_w_kernel" 2
run simt_f32 "cellmat_ffma" 1
run simt_f64 "cellmat_dmma" 1
run action "action_kernel" 1
run asm_p3 "assemble|cellmat_tc2" 4
python scripts/zoo_summary.py r2bt > $OUT/zoo_summary.txt 2>&1; echo "summary rc=$?"; cat $OUT/zoo_summary.txt
NCU_SUMMARY_DIR=$OUT python scripts/ncu_summary.py r2bt "$CMD" > /dev/null 2>&1; echo "launch summary rc=$?"
mkdir -p /tmp/ncu_keep
for f in $OUT/zoo_*.ncu-rep; do
  sz=$(stat -c %s "$f")
  if [ "$sz" -gt 12000000 ]; then mv "$f" /tmp/ncu_keep/; fi
done
ls -la $OUT | tail -30
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
