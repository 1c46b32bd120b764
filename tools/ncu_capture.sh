#!/bin/bash
# One GPU: launch list of 8 steady-state C2 ticks + full captures of the decode-attention kernel, a GEMM
# and the tcgen05 prefill/FT attention. Outputs land in gpurun_out/ (summarised into profiles/ by
# tools/summarize_ncu.py).
set -x
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python tools/profile_tick.py --steps 8 > gpurun_out/launch_run.log 2>&1
cp gpurun_out/decode_attn_bytes.json gpurun_out/decode_attn_bytes_launchlist.json
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode2 -s 12 -c 2 \
    -o gpurun_out/attn_decode python tools/profile_tick.py --steps 2 > gpurun_out/ncu_attn.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:gemm_tc_kernel -s 30 -c 3 \
    -o gpurun_out/gemm python tools/profile_tick.py --steps 2 > gpurun_out/ncu_gemm.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:attn_tc_kernel -s 2 -c 2 \
    -o gpurun_out/attn_tc python tools/profile_tick.py --steps 2 > gpurun_out/ncu_attn_tc.log 2>&1
ls -la gpurun_out
