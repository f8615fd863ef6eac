#!/bin/bash
# Build libwsort variants with different tile/merge geometries into build/variants/.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
build() {
  name=$1; shift
  out=build/variants/$name; mkdir -p $out
  for f in paper_1407_6603_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude "$@" -c $f -o $out/$b.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libwsort_b200.so $out/*.o
}
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  build $name $flags
done
