#!/bin/bash
# A/B of libchgpu variants (tools/build_variants.sh) with tools/knob_sweep.py.
cp paper_1508_05488_b200/libchgpu.so /tmp/orig.so
for rep in 1 2; do
echo -n "base "; timeout 300 python tools/knob_sweep.py X=0
for v in ${VARS:-ef fh both}; do cp build/variants/libchgpu_$v.so paper_1508_05488_b200/libchgpu.so; echo -n "$v "; timeout 300 python tools/knob_sweep.py X=0; done
cp /tmp/orig.so paper_1508_05488_b200/libchgpu.so
done
