#!/bin/bash
set -u
python scripts/k1_ab.py
for v in gw4 gw1; do MPFEM_B200_LIB=paper_2410_12614_b200/lib/diag/lib$v.so python scripts/k1_ab.py; done
