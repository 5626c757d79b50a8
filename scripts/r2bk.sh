#!/bin/bash
set -u
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cells.py tests/test_gpu_bounds.py tests/test_gpu_reference_suite.py -m gpu -x -q > $OUT/pytest_cells.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_cells.log
timeout 600 python scripts/kernel_zoo.py simt_f32 1 > $OUT/zoo_simt_f32.plain 2>&1 && timeout 900 ncu --set full --clock-control none -k "regex:cellmat_ffma" -c 1 -o $OUT/zoo_simt_f32 -f python scripts/kernel_zoo.py simt_f32 1 > $OUT/zoo_simt_f32.ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/zoo_simt_f32.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum 2>/dev/null | tail -2
