#!/bin/bash
# C1 (one 4096x4096 tensor) decode and the layer decode for a list of libs.
for l in $1; do
  NZGPU_LIB=$l python tools/quickbench.py 16777216 7,3,0 64 50 | sed "s/^/$l /"
  NZGPU_LIB=$l python tools/layerbench.py 7 30 64
done
