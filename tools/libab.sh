#!/bin/bash
# Interleaved A/B of decode-library variants on one box: for each round, run
# tools/layerbench.py once per library (NZGPU_LIB) and collect JSON lines.
# usage: tools/libab.sh "libnzgpu.so libnzgpu_x.so" "7,0" rounds [K]
libs=$1; precs=${2:-7}; rounds=${3:-3}; K=${4:-0}
for r in $(seq $rounds); do
  for l in $libs; do
    NZGPU_LIB=$l python tools/layerbench.py $precs 30 $K
  done
done
