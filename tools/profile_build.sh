#!/bin/bash
# Tree-build profile (under gpurun): launch list with DRAM bytes of the last of
# two 16M / 1M builds, and one --set full capture of k_subtrees at 16M.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for n in 16000000 1000000; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --csv --log-file gpurun_out/build_launches_$n.csv python tools/prof_build.py $n 2 > /dev/null 2>&1
  python tools/build_launches.py gpurun_out/build_launches_$n.csv > gpurun_out/build_table_$n.txt
done
ncu --set full --clock-control none --import-source on -k regex:k_subtrees -s 1 -c 1 -o gpurun_out/subtrees_full -f \
  python tools/prof_build.py 16000000 2 > /dev/null 2>&1
ncu -i gpurun_out/subtrees_full.ncu-rep --page raw --csv > gpurun_out/subtrees_raw.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/subtrees_full.ncu-rep 6 24 > gpurun_out/subtrees_hot.txt 2>&1
python tools/build_timing.py 1000000 16000000 > gpurun_out/build_timing.txt 2>&1
