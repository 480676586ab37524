#!/bin/bash
# One profiling pass for profiles/: plain run, launch list, full ncu capture of
# the hot kernels.  Run from the repo root on the GPU box (1 GPU).
set -u
OUT=gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-registration"
$CMD > $OUT/prof_bench_plain.json 2> $OUT/prof_bench_plain.err
echo "plain bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
python tools/prof_kernels.py --mode all --iters 2 > $OUT/prof_all_plain.log 2>&1
echo "prof plain rc=$?"
ncu --set full --clock-control none --import-source on \
    -k regex:"k_bh_iterate|k_direct_iterate32|k_gpe32" \
    -c 4 -o $OUT/full python tools/prof_kernels.py --mode all --iters 2 > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
python tools/prof_build.py 16000000 2 > $OUT/prof_build_plain.log 2>&1
echo "build plain rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
    --clock-control none --csv --log-file $OUT/build16m.csv python tools/prof_build.py 16000000 2 \
    > $OUT/ncu_build.log 2>&1
echo "build launch list rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
    --clock-control none --csv --log-file $OUT/build1m.csv python tools/prof_build.py 1000000 2 \
    > $OUT/ncu_build1m.log 2>&1
echo "build 1M launch list rc=$?"
