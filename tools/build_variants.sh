#!/bin/bash
# Library variants that differ in taylor.cu's compile-time knobs, for tools/ab_variants.sh:
#   tools/build_variants.sh name1 "flags1" name2 "flags2" ...   -> variants/lib<name>.so
set -e
P=paper_2603_07341_b200
PB200_KEEP_OBJS=1 python $P/build.py --force > /dev/null
mkdir -p variants
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC,-O2 -diag-suppress 177"
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  ( cd $P/csrc && nvcc $FLAGS $flags -c -o ../../variants/_taylor_$name.o taylor.cu )
  objs=$(ls $P/_*.o | grep -v _taylor.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib$name.so $objs variants/_taylor_$name.o -ldl
  rm variants/_taylor_$name.o
  echo "built variants/lib$name.so ($flags)"
done
rm -f $P/_*.o
