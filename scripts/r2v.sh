#!/bin/bash
set -u
timeout 300 python scripts/k12_time.py 2>&1
MPFEM_B200_LIB=paper_2410_12614_b200/lib/diag/libp1only.so timeout 300 python scripts/k12_time.py 2>&1 | grep "p=2 form=0"
timeout 900 python -m pytest tests/test_gpu_cells.py -m gpu -q -x -k "within_bound or full_config or batch or edge" 2>&1 | tail -2
