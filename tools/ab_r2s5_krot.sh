#!/bin/bash
# k-walk rotation of one-wave GEMMs: decode-sized shapes with cold weights, MACE_GEMM_KROT off / 1 / 5
set -x
SH="256,3072,2048,bf16 256,8192,2048,bf16_swiglu 256,2048,2048,f32_add 256,2048,8192,f32_add 256,128256,2048,f32 1215,2304,768,bf16 1215,768,3072,f32_add"
for k in 0 1 5; do
  MACE_GEMM_KROT=$k timeout 600 python tools/gemm_sweep.py --cold 8 --shapes $SH | sed "s/^/krot$k /"
done > gpurun_out/r2s5_krot_sweep.log 2>&1
MACE_GEMM_KROT=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "gemm" > gpurun_out/r2s5_krot_tests.log 2>&1
grep '^krot' gpurun_out/r2s5_krot_sweep.log | cut -c1-90; tail -2 gpurun_out/r2s5_krot_tests.log
