#!/bin/bash
# A/B helper (not part of the product): builds the library with extra nvcc
# flags into build/ab/lib<name>.so; select it at run time with CPRAND_LIB.
#   tools/build_variant.sh N1 -DCPB_COLD_FIT=__noinline__
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build/ab/$name
for f in paper_1701_06600_b200/csrc/*.cu; do
  o=build/ab/$name/$(basename ${f%.cu}).o
  (/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++20 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr "$@" -c $f -o $o 2> $o.log || (cat $o.log; exit 1)) &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/lib$name.so build/ab/$name/*.o -lnccl -lcudart
echo built build/ab/lib$name.so
