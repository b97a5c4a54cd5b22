#!/bin/bash
# dev A/B builds: recompile the given sources with extra flags and link them
# with the in-tree objects into dev/ab/libmmpr_<name>.so (MMPR_LIB=... to load)
# usage: dev/build_variant.sh <name> "<extra nvcc flags>" fine.cu [pipeline.cu ...]
set -e
name=$1; flags=$2; shift 2
C=paper_2310_11365_b200/csrc
mkdir -p dev/ab/$name
objs=""
for o in $C/build/*.o; do
  b=$(basename $o .o)
  skip=0
  for s in "$@"; do [ "$b" == "$(basename $s .cu)" ] && skip=1; done
  [ $skip == 0 ] && objs="$objs $o"
done
for s in "$@"; do
  b=$(basename $s .cu)
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -c $C/$s -o dev/ab/$name/$b.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o dev/ab/libmmpr_$name.so $objs dev/ab/$name/*.o -lcudart
echo built dev/ab/libmmpr_$name.so
