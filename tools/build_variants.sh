#!/bin/bash
# Builds libchgpu variants of one .cu file with extra -D flags:
#   tools/build_variants.sh k_filter "A:-DX=1 -DY=2" "B:-DX=2" ...
# -> build/variants/libchgpu_A.so ... (swap in place of paper_1508_05488_b200/libchgpu.so to A/B).
set -e
cd "$(dirname "$0")/.."
make -s >/dev/null
src=$1; shift
mkdir -p build/variants
others=$(ls build/*.o | grep -v "/$src" | grep -v "/api_" | grep -v acceptance)
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
    -Xcompiler -fPIC -Iinclude -Ipaper_1508_05488_b200/csrc $flags -c -o build/variants/$src.$name.o \
    paper_1508_05488_b200/csrc/$src.cu
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libchgpu_$name.so \
    build/variants/$src.$name.o $others -Xlinker -soname=libchgpu.so
  echo built $name
done
