#!/bin/bash
# A/B of the tcgen05 decode attention: one MMA issuer (MACE_DTC_ISSUE=1) vs split S / P.V issuers (default)
set -x
for i in 1 2 3; do
  MACE_DTC_ISSUE=1 timeout 300 python tools/decode_bench.py 2 128 32 8 256 1500 2 64 32 8 256 1920 2 128 32 8 64 2000 | sed 's/^/issue1 /'
  timeout 300 python tools/decode_bench.py 2 128 32 8 256 1500 2 64 32 8 256 1920 2 128 32 8 64 2000 | sed 's/^/split /'
done > gpurun_out/r2s5_dtc_ab3.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "attn or decode or attention or c1 or families" > gpurun_out/r2s5_dtc_tests3.log 2>&1
grep '^issue1\|^split' gpurun_out/r2s5_dtc_ab3.log | cut -c1-200; tail -2 gpurun_out/r2s5_dtc_tests3.log
