#!/bin/bash
# ncu --set full captures of the hot kernels on bench.py's configs[2] workload
# (one launch each, first force pass = the initial state), into gpurun_out/.
# Run under gpurun only after the plain command exited 0.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -c 1"
$NCU -k regex:k_bh_iterate -s 2 -o gpurun_out/bh_full -f python tools/prof_kernels.py --mode bh --iters 3 > gpurun_out/ncu_bh.log 2>&1
$NCU -k regex:k_gpe32 -o gpurun_out/gpe_full -f python tools/prof_kernels.py --mode gpe --iters 1 > gpurun_out/ncu_gpe.log 2>&1
$NCU -k regex:k_bh_operator -o gpurun_out/op_full -f python tools/e2e_timing.py 1 > gpurun_out/ncu_op.log 2>&1
for r in bh gpe op; do ncu -i gpurun_out/${r}_full.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null; done
ncu -i gpurun_out/bh_full.ncu-rep --page source --csv --print-source sass > gpurun_out/bh_source.csv 2>/dev/null
echo done
