#!/bin/bash
# K2 bin-max sampling (CHGPU_FILTER_WSAMPLE_LOG2) per distribution.
for d in uniform_square uniform_disk gaussian circle; do
  for k in 0 1 2; do
    echo -n "$d ws$k "; DIST=$d timeout 300 python tools/knob_sweep.py CHGPU_FILTER_WSAMPLE_LOG2=$k
  done
done
