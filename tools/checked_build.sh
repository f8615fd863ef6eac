#!/bin/bash
# Checked build of the library (WS_CHECKED=1: device bounds checks on every
# computed shared / global index, ws_debug_checks() reads them) into
# build/checked/libwsort_b200.so. Run the GPU suite against it with
#   WSORT_LIB=$PWD/build/checked/libwsort_b200.so WSORT_CHECKED=1 python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/.."
out=build/checked
mkdir -p $out
for f in paper_1407_6603_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
       -DWS_CHECKED=1 -c $f -o $out/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libwsort_b200.so $out/*.o
echo "checked build: $out/libwsort_b200.so"
