set -u
mkdir -p gpurun_out
for lib in "" paper_2410_12614_b200/lib/diag/libmpfem_b200_nomma.so; do
for ov in 1 0; do echo "lib=$lib ov=$ov"; MPFEM_B200_LIB=$lib MPFEM_B200_OVERLAP=$ov timeout 100 python scripts/trace_overlap.py | tail -1; done
done
