#!/bin/bash
set -u
for i in 1 2; do
echo "shipped"; timeout 400 python scripts/modes_ab.py 2>&1 | tail -1
echo "bulk"; MPFEM_B200_LIB=$PWD/paper_2410_12614_b200/lib/diag/libbulk.so timeout 400 python scripts/modes_ab.py 2>&1 | tail -1
done
