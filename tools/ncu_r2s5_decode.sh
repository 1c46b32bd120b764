#!/bin/bash
# Source-level ncu captures of the tcgen05 decode attention (hd 128 C4 shape, hd 64 C3 shape) in the
# microbenchmark; outputs gpurun_out/r2s5_dtc*.ncu-rep
set -x
python tools/decode_bench.py 2 128 32 8 256 1500 2 64 32 8 256 1920 > gpurun_out/r2s5_decode_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode_tc -s 3 -c 1 \
    -o gpurun_out/r2s5_dtc128 python tools/decode_bench.py 2 128 32 8 256 1500 > gpurun_out/r2s5_ncu_dtc128.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode_tc -s 3 -c 1 \
    -o gpurun_out/r2s5_dtc64 python tools/decode_bench.py 2 64 32 8 256 1920 > gpurun_out/r2s5_ncu_dtc64.log 2>&1
cat gpurun_out/r2s5_decode_bench.log; ls -la gpurun_out/*.ncu-rep
