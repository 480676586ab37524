# Round-end check on one B200 (run through gpurun from the repo root):
# the GPU test suite, the default bench line and smoke(), logs under gpurun_out/.
mkdir -p gpurun_out; timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/full_tests.log 2>&1; echo "rc=$?" >> gpurun_out/full_tests.log; timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/full_tests.log; timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/full_tests.log 2>&1
