#!/bin/bash
# tools/build_variant.sh NAME "EXTRA NVCC FLAGS" [alternative rtk_kernels.cu]
# Builds ab/NAME/paper_2501_14336_b200 (python package + librtk_b200.so) where rtk_kernels.cu is
# recompiled with the extra flags (other objects reused from the in-tree build); for same-box
# A/B runs (tools/ab_*.py take the package's parent directory). ab/ is git-ignored.
set -e
R=/root/repo; N=$1; F=$2; SRC=${3:-$R/paper_2501_14336_b200/csrc/rtk_kernels.cu}
D=$R/ab/$N/paper_2501_14336_b200
rm -rf $R/ab/$N; mkdir -p $D/build
cp $R/paper_2501_14336_b200/*.py $D/
cp $SRC $R/paper_2501_14336_b200/csrc/_variant_kernels.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 $F \
  -c $R/paper_2501_14336_b200/csrc/_variant_kernels.cu -o $D/build/rtk_kernels.o
rm -f $R/paper_2501_14336_b200/csrc/_variant_kernels.cu
objs=""; for o in $R/paper_2501_14336_b200/build/*.o; do b=$(basename $o); [ $b = rtk_kernels.o ] || objs="$objs $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/librtk_b200.so $D/build/rtk_kernels.o $objs -lcudart_static -lrt -lpthread -ldl
rm -rf $D/build; echo "built $D"
