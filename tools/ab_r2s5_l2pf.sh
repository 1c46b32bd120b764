#!/bin/bash
# L2 prefetch of the weight boxes ahead of the TMA ring: decode-sized shapes with cold weights, MACE_GEMM_L2PF 0/8/16/24
set -x
SH="256,3072,2048,bf16 256,8192,2048,bf16_swiglu 256,2048,2048,f32_add 256,2048,8192,f32_add 256,128256,2048,f32 1215,2304,768,bf16 1215,768,3072,f32_add 8192,4096,4096,bf16"
for k in 0 8 16 24; do
  MACE_GEMM_L2PF=$k timeout 600 python tools/gemm_sweep.py --cold 8 --shapes $SH | sed "s/^/pf$k /"
done > gpurun_out/r2s5_l2pf_sweep.log 2>&1
MACE_GEMM_L2PF=16 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "gemm" > gpurun_out/r2s5_l2pf_tests.log 2>&1
grep '^pf' gpurun_out/r2s5_l2pf_sweep.log | cut -c1-80; tail -2 gpurun_out/r2s5_l2pf_tests.log
