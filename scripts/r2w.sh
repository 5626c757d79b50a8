#!/bin/bash
set -u
python scripts/k1_ab.py
timeout 300 python scripts/k12_time.py 2>&1 | head -12
timeout 900 python -m pytest tests/test_gpu_cells.py tests/test_gpu_box.py -m gpu -q -x 2>&1 | tail -3
