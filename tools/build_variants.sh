#!/bin/bash
# Builds libchgpu variants with extra -D flags, for A/B timing on the GPU box:
#   tools/build_variants.sh <src|ALL> "A:-DX=1 -DY=2" "B:-DX=2" ...
# <src> (e.g. k_filter) recompiles that one .cu; ALL recompiles every .cu.
# -> build/variants/libchgpu_A.so ... (CHGPU_LIB=build/variants/libchgpu_A.so selects one).
set -e
cd "$(dirname "$0")/.."
make -s >/dev/null
src=$1; shift
mkdir -p build/variants
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_1508_05488_b200/csrc"
CU="k_discard k_sort k_spa k_filter k_convex pipeline"
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  if [ "$src" = ALL ]; then redo=$CU; else redo=$src; fi
  objs=""
  for c in $CU; do
    if echo " $redo " | grep -q " $c "; then
      $NV $FL $flags -c -o build/variants/$c.$name.o paper_1508_05488_b200/csrc/$c.cu
      objs="$objs build/variants/$c.$name.o"
    else
      objs="$objs build/$c.o"
    fi
  done
  $NV -shared -o build/variants/libchgpu_$name.so $objs build/finisher.o build/datasets.o \
    -Xlinker -soname=libchgpu.so
  echo built $name
done
