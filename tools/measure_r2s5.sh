#!/bin/bash
# Round-2 session-5 check of the rebuilt tree on one GPU (outputs gpurun_out/r2s5_*).
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s5_gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s5_smoke.log 2>&1
python bench.py > gpurun_out/r2s5_bench_c4.log 2>&1
tail -2 gpurun_out/r2s5_gpu_tests.log; tail -1 gpurun_out/r2s5_smoke.log
tail -c 400 gpurun_out/r2s5_bench_c4.log
