#!/bin/bash
# GEMM CTAs exit after the stores' smem reads (not the write round trip): trace, tests, C2 / C3 / C4 lines
set -x
python tools/gemm_trace.py 1215 2304 768 bf16 2>&1 | tail -10 > gpurun_out/r2s5_tail_trace.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s5_tail_tests.log 2>&1
python bench.py --workload c2 > gpurun_out/r2s5_tail_bench_c2.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s5_tail_bench_c3.log 2>&1
python bench.py > gpurun_out/r2s5_tail_bench_c4.log 2>&1
cat gpurun_out/r2s5_tail_trace.log; tail -2 gpurun_out/r2s5_tail_tests.log
