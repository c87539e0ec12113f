#!/bin/bash
# tools/build_variant.sh NAME FILE.cu "EXTRA NVCC FLAGS" [alternative source for FILE.cu]
# Builds ab/NAME/paper_2501_14336_b200 (python package + librtk_b200.so) with csrc/FILE.cu
# recompiled with the extra flags (other objects reused from the in-tree build), for same-box A/B
# runs (tools/ab_*.py take the package's parent directory). ab/ is git-ignored; delete it before
# gpurun calls that do not need it (it travels with the snapshot).
set -e
R=/root/repo; N=$1; FILE=$2; F=$3; SRC=${4:-$R/paper_2501_14336_b200/csrc/$FILE}
D=$R/ab/$N/paper_2501_14336_b200
rm -rf $R/ab/$N; mkdir -p $D/build
cp $R/paper_2501_14336_b200/*.py $D/
cp $SRC $R/paper_2501_14336_b200/csrc/_variant.cu
B=$(basename $FILE .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 $F \
  -c $R/paper_2501_14336_b200/csrc/_variant.cu -o $D/build/$B.o 2>/dev/null
rm -f $R/paper_2501_14336_b200/csrc/_variant.cu
objs=""; for o in $R/paper_2501_14336_b200/build/*.o; do b=$(basename $o); [ $b = $B.o ] || objs="$objs $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/librtk_b200.so $D/build/$B.o $objs -lcudart_static -lrt -lpthread -ldl
rm -rf $D/build; echo "built $D"
