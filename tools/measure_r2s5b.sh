#!/bin/bash
# Benches after the decode-attention producer change (outputs gpurun_out/r2s5b_*)
set -x
python bench.py > gpurun_out/r2s5b_bench_c4.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s5b_bench_c3.log 2>&1
python tools/tick_split.py c3 > gpurun_out/r2s5b_tick_split_c3.log 2>&1
python bench.py --workload c2 > gpurun_out/r2s5b_bench_c2.log 2>&1
for f in c4 c3 c2; do tail -c 300 gpurun_out/r2s5b_bench_$f.log; echo; done
tail -3 gpurun_out/r2s5b_tick_split_c3.log
