#!/bin/bash
# MHA (GPT-2, G = 1) decode attention: CUDA-core streaming kernel (impl 1) vs tcgen05 swap-AB (impl 2) after the
# tcgen05 producer change; microbench shapes + the C2 bench line with each (outputs gpurun_out/r2s5_mha_*)
set -x
for i in 1 2; do
  timeout 300 python tools/decode_bench.py 1 64 12 12 200 400 2 64 12 12 200 400 1 64 12 12 256 800 2 64 12 12 256 800 1 64 12 12 64 300 2 64 12 12 64 300
done > gpurun_out/r2s5_mha_micro.log 2>&1
MACE_DECODE_IMPL=2 timeout 600 python bench.py --workload c2 > gpurun_out/r2s5_mha_bench_c2_impl2.log 2>&1
MACE_DECODE_IMPL=1 timeout 600 python bench.py --workload c2 > gpurun_out/r2s5_mha_bench_c2_impl1.log 2>&1
grep '^{' gpurun_out/r2s5_mha_micro.log | cut -c1-150
for f in impl2 impl1; do tail -c 200 gpurun_out/r2s5_mha_bench_c2_$f.log; echo; done
