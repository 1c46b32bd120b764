#!/bin/bash
# in-kernel phase traces of the C2 / C3 one-wave projection GEMMs (single-CTA kernel, auto tile choice)
for s in "1215 2304 768 bf16" "1215 3072 768 bf16_gelu" "1215 768 768 f32_add" "256 3072 2048 bf16" "256 2048 2048 f32_add" "1215 3072 768 bf16"; do
  echo "== $s"; python tools/gemm_trace.py $s 2>&1 | tail -12
done > gpurun_out/r2s5_trace_c2c3.log 2>&1
cat gpurun_out/r2s5_trace_c2c3.log
