#!/bin/bash
# Round-2 captures on one GPU (outputs gpurun_out/r2_*; summarised by tools/summarize_ncu.py profiles r2):
#   launch list of 2 C4 fine-tune-carrying ticks (the bench's timed window starts at tick 8)
#   --set full: masked AdamW (float4 kernel, C4 top-2 layers, 436M parameters), the KV paging kernels
#   (decode_alloc / trim / release / page_copy / set_tables, C2 steady state), the C4 CTA-pair GEMM.
set -x
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_c4_launches.csv python tools/profile_tick.py --workload c4 --skip 8 --steps 2 \
    > gpurun_out/r2_launch_c4.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:adamw -c 1 \
    -o gpurun_out/adamw python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2_ncu_adamw.log 2>&1
ncu --profile-from-start off --set full --clock-control none \
    -k regex:"decode_alloc|trim_kernel|release_kernel|page_copy|set_tables|bump_end|reset_slot" -c 12 \
    -o gpurun_out/paging python tools/profile_tick.py --workload c2 --steps 4 > gpurun_out/r2_ncu_paging.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:gemm_tc2_kernel -s 10 -c 2 \
    -o gpurun_out/gemm_pair python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2_ncu_gemm2.log 2>&1
ls -la gpurun_out/*.ncu-rep
