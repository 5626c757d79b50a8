#!/bin/bash
# Round-2z GPU session: source-level ncu of the mass K1 (config 0) and of the fused small-p kernel;
# reports are processed on the box (they embed the whole cubin and exceed the copy-back limit).
set -u
OUT=gpurun_out
mkdir -p $OUT /tmp/ncu_keep
rm -f $OUT/*.ncu-rep
run() {  # kind regex count
  local kind=$1 re=$2 cnt=$3
  timeout 600 python scripts/kernel_zoo.py $kind 1 > $OUT/zoo_$kind.plain 2>&1 || { echo "$kind plain FAILED"; tail -3 $OUT/zoo_$kind.plain; return; }
  timeout 1200 ncu --set full --clock-control none -k "regex:$re" -c $cnt \
    -o /tmp/ncu_keep/zoo_$kind -f python scripts/kernel_zoo.py $kind 1 > $OUT/zoo_$kind.ncu.log 2>&1
  echo "$kind ncu rc=$?"
  ncu -i /tmp/ncu_keep/zoo_$kind.ncu-rep --page raw --csv > $OUT/zoo_$kind.raw.csv 2>/dev/null
}
OBJ=paper_2410_12614_b200/lib/obj
run mass_k2 "geom_w_kernel" 1
python scripts/ncu_lines.py /tmp/ncu_keep/zoo_mass_k2.ncu-rep $OBJ/launch_geom.o _ZN10mpfem_b20013geom_w_kernelI6__halfLi2ELi1ELi1EEEvNS_11GeomWParamsE 8192 > $OUT/lines_mass_k1.txt 2>&1
run fused_p1 "fused" 1
FN=$(cuobjdump -elf $OBJ/launch_fused.o 2>/dev/null | grep -o "_ZN[A-Za-z0-9_]*fused[A-Za-z0-9_]*" | sort -u | head -40 > $OUT/fused_syms.txt; true)
ls -la $OUT | tail
