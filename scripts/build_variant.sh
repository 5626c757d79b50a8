#!/bin/bash
# usage: build_variant.sh NAME "-DFLAGS..."  -> paper_2410_12614_b200/lib/diag/libNAME.so
set -e
cd /root/repo
NAME=$1; shift
OUT=/tmp/var_$NAME; rm -rf $OUT; mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr $*"
for f in capi launch_geom launch_fused assembly_capi launch_geom_box launch_action geom_tensor assembly_host; do $NV -c -o $OUT/$f.o paper_2410_12614_b200/csrc/$f.cu & done
wait
mkdir -p paper_2410_12614_b200/lib/diag
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2410_12614_b200/lib/diag/lib$NAME.so $OUT/*.o paper_2410_12614_b200/lib/obj/launch_bounds.o paper_2410_12614_b200/lib/obj/host_setup.o paper_2410_12614_b200/lib/obj/host_mesh.o
echo built lib$NAME.so
