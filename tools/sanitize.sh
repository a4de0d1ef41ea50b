#!/bin/bash
# compute-sanitizer over the codec's kernels (tools/sanitize_run.py, small
# inputs), both decode schedules, plus the drop-in C++ suite under memcheck.
# Logs go to gpurun_out/sanitize_*.log; the last line of each is the
# sanitizer's summary ("ERROR SUMMARY: N errors").
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for kern in persist tiles; do
    NZGPU_KERNEL=$kern timeout 1200 $CS --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_run.py 100000 > gpurun_out/sanitize_${tool}_${kern}.log 2>&1
    echo "$tool $kern rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${kern}.log | tail -1)"
  done
done
g++ -std=c++20 -O2 -pthread -I include tests/cpp/dropin_test.cpp -L paper_2410_20650_b200 -lnzgpu \
  -Wl,-rpath,$PWD/paper_2410_20650_b200 -o build/dropin_test_san && \
  timeout 1800 $CS --tool memcheck build/dropin_test_san > gpurun_out/sanitize_memcheck_dropin.log 2>&1
echo "memcheck dropin rc=$? $(grep -h 'ERROR SUMMARY' gpurun_out/sanitize_memcheck_dropin.log | tail -1)"
