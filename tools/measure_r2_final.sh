#!/bin/bash
# Round-2 final measurements on one GPU (outputs gpurun_out/r2f_*): the GPU suite, smoke, the default bench (C4)
# and its reference arm, C3 / C2 bench lines, C3 / C2 tick splits.
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f_gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
python bench.py > gpurun_out/r2f_bench_c4.log 2>&1
python bench.py --impl reference > gpurun_out/r2f_bench_c4_reference.log 2>&1
python bench.py --workload c3 > gpurun_out/r2f_bench_c3.log 2>&1
python bench.py --workload c2 > gpurun_out/r2f_bench_c2.log 2>&1
python tools/tick_split.py c3 > gpurun_out/r2f_tick_split_c3.log 2>&1
python tools/tick_split.py c2 > gpurun_out/r2f_tick_split_c2.log 2>&1
tail -2 gpurun_out/r2f_gpu_tests.log; tail -1 gpurun_out/r2f_smoke.log
for f in c4 c4_reference c3 c2; do tail -c 300 gpurun_out/r2f_bench_$f.log; echo; done
tail -3 gpurun_out/r2f_tick_split_c3.log gpurun_out/r2f_tick_split_c2.log
