#!/bin/bash
# SwiGLU epilogue with the branch-free reciprocal: trace, sweep (decode-sized + prefill-sized), swiglu / family
# parity tests, C3 / C4 bench lines (outputs gpurun_out/r2s5_sw_*)
set -x
MACE_GEMM_FORCE=single python tools/gemm_trace.py 256 16384 2048 bf16_swiglu > gpurun_out/r2s5_sw_trace.log 2>&1
python tools/gemm_sweep.py --cold 8 --shapes 256,8192,2048,bf16_swiglu 512,8192,2048,bf16_swiglu 1024,8192,2048,bf16_swiglu 4096,14336,4096,bf16_swiglu 16384,14336,4096,bf16_swiglu 256,16384,2048,bf16 > gpurun_out/r2s5_sw_sweep.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "gemm or families or c1 or lora" > gpurun_out/r2s5_sw_tests.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s5_sw_bench_c3.log 2>&1
python tools/tick_split.py c3 > gpurun_out/r2s5_sw_tick_split_c3.log 2>&1
python bench.py > gpurun_out/r2s5_sw_bench_c4.log 2>&1
tail -4 gpurun_out/r2s5_sw_trace.log; grep "M=" gpurun_out/r2s5_sw_sweep.log | cut -c1-90; tail -2 gpurun_out/r2s5_sw_tests.log
tail -2 gpurun_out/r2s5_sw_tick_split_c3.log
for f in c3 c4; do tail -c 250 gpurun_out/r2s5_sw_bench_$f.log; echo; done
