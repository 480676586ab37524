#!/bin/bash
# Round profile set (run under gpurun after a clean plain bench run):
#   gpurun_out/launches_bench.csv  ncu launch list of a short bench.py run
#   gpurun_out/{bh,gpe}_full.ncu-rep + *_raw.csv + bh_source.csv (tools/profile_kernels.sh)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-registration --no-configs0 \
  --no-configs --no-ingest --no-build > gpurun_out/ncu_bench.log 2>&1
bash tools/profile_kernels.sh
