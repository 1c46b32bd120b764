#!/bin/bash
# ncu --set full of the decode-sized (M = 256) projections of C3: SwiGLU up (pair kernel), qkv, o, down, lm_head
# (cold weights: ncu flushes the caches between replays). Outputs gpurun_out/r2s5_gemm_*.ncu-rep
set -x
P="ncu --set full --import-source on --clock-control none"
$P -k regex:gemm -s 2 -c 1 -o gpurun_out/r2s5_gemm_swiglu python tools/gemm_one.py 256 16384 2048 bf16_swiglu 3 > gpurun_out/r2s5_ncu_gemm_swiglu.log 2>&1
$P -k regex:gemm -s 2 -c 1 -o gpurun_out/r2s5_gemm_qkv python tools/gemm_one.py 256 3072 2048 bf16 3 > gpurun_out/r2s5_ncu_gemm_qkv.log 2>&1
$P -k regex:gemm -s 2 -c 1 -o gpurun_out/r2s5_gemm_lmhead python tools/gemm_one.py 256 128256 2048 f32 3 > gpurun_out/r2s5_ncu_gemm_lmhead.log 2>&1
python tools/gemm_sweep.py --cold 8 --shapes 256,3072,2048,bf16 256,8192,2048,bf16_swiglu 256,2048,8192,f32_add 256,128256,2048,f32 > gpurun_out/r2s5_gemm_sweep_cold.log 2>&1
ls -la gpurun_out/r2s5_gemm_*; cat gpurun_out/r2s5_gemm_sweep_cold.log | tail -5
