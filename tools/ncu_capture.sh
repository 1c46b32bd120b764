#!/bin/bash
# One GPU: launch lists of 8 steady-state C2 ticks and 2 C4 ticks, plus --set full captures of the top kernels:
# decode attention (C2 MHA CUDA-core kernel, C3 GQA tcgen05 kernel), the single-CTA GEMM (C2), the CTA-pair GEMM
# (C4) and the warp-specialised prefill/FT attention (C2 hd 64, C4 hd 128). Outputs land in gpurun_out/
# (summarised into profiles/ by tools/summarize_ncu.py).
set -x
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python tools/profile_tick.py --steps 8 > gpurun_out/launch_run.log 2>&1
cp gpurun_out/decode_attn_bytes.json gpurun_out/decode_attn_bytes_launchlist.json
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode2 -s 12 -c 2 \
    -o gpurun_out/attn_decode python tools/profile_tick.py --steps 2 > gpurun_out/ncu_attn.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:gemm_tc_kernel -s 30 -c 3 \
    -o gpurun_out/gemm python tools/profile_tick.py --steps 2 > gpurun_out/ncu_gemm.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_fa_kernel -s 2 -c 2 \
    -o gpurun_out/attn_fa python tools/profile_tick.py --steps 2 > gpurun_out/ncu_attn_fa.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:attn_decode_tc -s 4 -c 2 \
    -o gpurun_out/attn_decode_tc python tools/profile_tick.py --workload c3 --steps 2 > gpurun_out/ncu_attn_dtc.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4.csv python tools/profile_tick.py --workload c4 --steps 2 > gpurun_out/launch_c4.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:gemm_tc2_kernel -s 10 -c 2 \
    -o gpurun_out/gemm_pair python tools/profile_tick.py --workload c4 --steps 1 > gpurun_out/ncu_gemm2.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:attn_fa_kernel -s 4 -c 1 \
    -o gpurun_out/attn_fa_c4 python tools/profile_tick.py --workload c4 --steps 1 > gpurun_out/ncu_attn_fa4.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:attn_bwd_tc -s 0 -c 1 \
    -o gpurun_out/attn_bwd_c4 python tools/profile_tick.py --workload c4 --steps 1 > gpurun_out/ncu_attn_bwd4.log 2>&1
ls -la gpurun_out
