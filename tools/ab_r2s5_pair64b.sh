#!/bin/bash
# tile policy with CTA-pair BN 64: GPU suite + C3 / C2 / C4 lines
set -x
python tools/gemm_sweep.py --cold 8 --shapes 256,2048,2048,f32_add 600,768,3072,f32_add 1215,768,3072,f32_add 256,3072,2048,bf16 > gpurun_out/r2s5_pair64b_sweep.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s5_pair64b_tests.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s5_pair64b_bench_c3.log 2>&1
python tools/tick_split.py c3 > gpurun_out/r2s5_pair64b_tick_split_c3.log 2>&1
python bench.py --workload c2 > gpurun_out/r2s5_pair64b_bench_c2.log 2>&1
python bench.py > gpurun_out/r2s5_pair64b_bench_c4.log 2>&1
grep "M=" gpurun_out/r2s5_pair64b_sweep.log | cut -c1-80; tail -2 gpurun_out/r2s5_pair64b_tests.log; tail -3 gpurun_out/r2s5_pair64b_tick_split_c3.log
