#!/bin/bash
# Round-2 session-2 captures on one GPU (outputs gpurun_out/r2s2_*): the C4 launch list of 2 fine-tune ticks of the
# bench window, and --set full captures of the C4 row kernels (rope_kv, norm), C4 decode / prefill / backward
# attention, and C2's decode attention and single-CTA GEMM.
set -x
P="ncu --profile-from-start off --clock-control none"
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s2_c4_launches.csv \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 2 > gpurun_out/r2s2_launch_c4.log 2>&1
$P --set full --import-source on -k regex:"rope_kv|norm_wide" -s 20 -c 2 -o gpurun_out/r2s2_rows_c4 \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2s2_ncu_rows.log 2>&1
$P --set full --import-source on -k regex:attn_decode_tc -s 4 -c 1 -o gpurun_out/r2s2_dtc_c4 \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2s2_ncu_dtc.log 2>&1
$P --set full --import-source on -k regex:attn_fa_kernel -s 4 -c 1 -o gpurun_out/r2s2_fa_c4 \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2s2_ncu_fa.log 2>&1
$P --set full --import-source on -k regex:attn_bwd_tc -s 0 -c 1 -o gpurun_out/r2s2_bwd_c4 \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2s2_ncu_bwd.log 2>&1
$P --set full --import-source on -k regex:attn_decode2 -s 12 -c 1 -o gpurun_out/r2s2_dec_c2 \
   python tools/profile_tick.py --steps 2 > gpurun_out/r2s2_ncu_dec2.log 2>&1
$P --set full --import-source on -k regex:gemm_tc_kernel -s 30 -c 3 -o gpurun_out/r2s2_gemm_c2 \
   python tools/profile_tick.py --steps 2 > gpurun_out/r2s2_ncu_gemm_c2.log 2>&1
python tools/ft_diag.py 2 > gpurun_out/r2s2_ft_diag.log 2>&1
ls -la gpurun_out
