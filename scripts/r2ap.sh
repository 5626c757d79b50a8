#!/bin/bash
set -u
for v in pullC25 pullC50 pullC75 pullD25 pullD50 pullD75 pullB50; do MPFEM_B200_LIB=$PWD/paper_2410_12614_b200/lib/diag/lib$v.so timeout 600 python scripts/pull_time.py 2 3; done
