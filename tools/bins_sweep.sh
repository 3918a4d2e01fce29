#!/bin/bash
# SPA bins per chunk x bin-max sampling, 20M uniform and disk.
for d in uniform_square uniform_disk; do
for b in 7 8 9; do for w in 1 2; do
  echo -n "$d b$b w$w "; DIST=$d timeout 300 python tools/knob_sweep.py "CHGPU_FILTER_BINS_PER_CHUNK_LOG2=$b CHGPU_FILTER_WSAMPLE_LOG2=$w"
done; done; done
