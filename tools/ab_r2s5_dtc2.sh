#!/bin/bash
# decode attention, producer-only next-item lookahead: microbench (GQA + MHA on the tcgen05 kernel) + parity tests
set -x
for i in 1 2; do
  timeout 300 python tools/decode_bench.py 2 128 32 8 256 1500 2 64 32 8 256 1920 2 128 32 8 64 2000 2 64 12 12 200 400 2 64 12 12 64 300 2 128 32 8 256 600
done > gpurun_out/r2s5_dtc_ab4.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "attn or decode or attention or c1 or families" > gpurun_out/r2s5_dtc_tests4.log 2>&1
grep '^{' gpurun_out/r2s5_dtc_ab4.log | cut -c1-160; tail -2 gpurun_out/r2s5_dtc_tests4.log
