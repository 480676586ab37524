#!/bin/bash
# Build libfga with the device-side invariant checks (FGA_CHECKS=1) and run
# the GPU suite's race-prone subsets against it (under gpurun):
#   bash tools/check_build.sh [build|run]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
if [ "${1:-build}" = "build" ]; then
  tools/build_variant.sh checks "-DFGA_CHECKS=1"
else
  FGA_LIB_PATH=$PWD/paper_2009_14005_b200/_lib/libfga_checks.so python -m pytest -q -m gpu \
    tests/test_gpu_determinism.py tests/test_gpu_operators.py tests/test_gpu_batched.py \
    tests/test_gpu_register.py tests/test_gpu_regressions.py tests/test_gpu_two_d.py \
    tests/test_gpu_teacher_forced.py 2>&1 | tail -3
fi
