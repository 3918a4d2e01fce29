#!/bin/bash
# K2 variants: timing (tools/abl_k2.sh), then the filter-path parity tests
# with the first variant swapped in.
VARS="${VARS:-sk sk5}" bash tools/abl_k2.sh
for d in uniform_disk gaussian; do
  for v in base ${VARS:-sk sk5}; do
    [ $v != base ] && cp build/variants/libchgpu_$v.so paper_1508_05488_b200/libchgpu.so
    echo -n "$d $v "; DIST=$d timeout 300 python tools/knob_sweep.py X=0
    cp /tmp/orig.so paper_1508_05488_b200/libchgpu.so
  done
done
first=$(echo ${VARS:-sk sk5} | cut -d' ' -f1)
cp build/variants/libchgpu_$first.so paper_1508_05488_b200/libchgpu.so
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/k2v_pytest.log 2>&1; echo "pytest($first)=$?"; tail -2 gpurun_out/k2v_pytest.log
cp /tmp/orig.so paper_1508_05488_b200/libchgpu.so
