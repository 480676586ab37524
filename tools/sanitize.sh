#!/bin/bash
# compute-sanitizer over the race-prone kernels, one tool per call:
#   bash tools/sanitize.sh racecheck|synccheck|memcheck|initcheck
# Cases: the tree build's block-boundary tests (k_subtrees: barrier-free
# last-arriver climb over byte-packed shared counters; k_hier/k_crossing),
# small batched registrations (k_register_batch: shared-memory trees,
# windows under __syncwarp), a config-1 registration (k_bh_iterate with the
# shared fold sums, reductions, update) and the operators.  Logs ->
# gpurun_out/sanitize_<tool>.log
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TOOL=${1:-memcheck}
EXTRA=""
[ "$TOOL" = "racecheck" ] && EXTRA="--racecheck-report all"
compute-sanitizer --tool "$TOOL" $EXTRA --print-limit 50 --error-exitcode 9 \
  python -m pytest -q -m gpu -p no:cacheprovider \
    "tests/test_gpu_operators.py::test_tree_build_block_boundaries" \
    "tests/test_gpu_batched.py::test_batch_reports_per_pair_failures" \
    "tests/test_gpu_register.py::test_register_matches_reference_c1[fp32-0]" \
    "tests/test_gpu_operators.py::test_bh_forces_fp32_exact_visits" \
    "tests/test_gpu_regressions.py::test_theta_zero_with_shared_depth_cap_leaves" \
  > gpurun_out/sanitize_${TOOL}.log 2>&1
rc=$?
echo "compute-sanitizer $TOOL exit $rc" | tee -a gpurun_out/sanitize_${TOOL}.log
tail -5 gpurun_out/sanitize_${TOOL}.log
