#!/bin/bash
# The GPU test suite against the bounds-checked build of the library
# (NZ_CHECKS=1: device-side asserts on every output store, shared-memory
# window read and encoder scratch write; a violation traps the launch).
# Stand-in for compute-sanitizer, which is closed on this GPU pool.
# usage (GPU box): tools/checked_suite.sh > gpurun_out/checked_suite.log
python paper_2410_20650_b200/_build.py --define NZ_CHECKS=1 --out libnzgpu_checks.so > /dev/null || exit 1
NZGPU_LIB=libnzgpu_checks.so timeout 1800 python -m pytest tests -m gpu -q -x \
  --deselect tests/test_gpu_acceptance.py --deselect tests/test_gpu_cli.py --deselect tests/test_cpp_dropin.py \
  -p no:randomly
echo "checked suite rc=$?"
