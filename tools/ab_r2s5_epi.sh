#!/bin/bash
# GEMM epilogue staging: st.shared, plain fast path, vectorised bias chunks (outputs gpurun_out/r2s5_epi2_*)
set -x
for s in "1215 2304 768 bf16" "1215 768 768 f32_add" "256 3072 2048 bf16"; do echo "== $s"; python tools/gemm_trace.py $s 2>&1 | tail -15; done > gpurun_out/r2s5_epi2_trace.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s5_epi2_tests.log 2>&1
python bench.py --workload c2 > gpurun_out/r2s5_epi2_bench_c2.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s5_epi2_bench_c3.log 2>&1
python tools/tick_split.py c3 > gpurun_out/r2s5_epi2_tick_split_c3.log 2>&1
python bench.py > gpurun_out/r2s5_epi2_bench_c4.log 2>&1
grep -E "==|t0_epi_end|last_grp|epi_loop_done_w4|exit" gpurun_out/r2s5_epi2_trace.log; tail -2 gpurun_out/r2s5_epi2_tests.log; tail -2 gpurun_out/r2s5_epi2_tick_split_c3.log
