#!/bin/bash
# Round-2 session-4 measurements on one GPU (outputs gpurun_out/r2s4_*): the default bench (C4) and its reference arm,
# C3 / C2 bench lines (whole-tick roofline), the C2 launch list, and --set full captures of C2's decode attention
# and projection GEMMs.
set -x
python bench.py > gpurun_out/r2s4_bench_c4.log 2>&1
python bench.py --impl reference > gpurun_out/r2s4_bench_c4_reference.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s4_bench_c3.log 2>&1
python bench.py --workload c2 > gpurun_out/r2s4_bench_c2.log 2>&1
P="ncu --profile-from-start off --clock-control none"
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s4_c2_launches.csv \
   python tools/profile_tick.py --workload c2 --steps 16 > gpurun_out/r2s4_launch_c2.log 2>&1
$P --set full --import-source on -k regex:attn_decode2 -s 12 -c 1 -o gpurun_out/r2s4_dec_c2 \
   python tools/profile_tick.py --steps 2 > gpurun_out/r2s4_ncu_dec2.log 2>&1
$P --set full --import-source on -k regex:gemm_tc -s 30 -c 4 -o gpurun_out/r2s4_gemm_c2 \
   python tools/profile_tick.py --steps 2 > gpurun_out/r2s4_ncu_gemm_c2.log 2>&1
for f in gpurun_out/r2s4_bench_c4.log gpurun_out/r2s4_bench_c4_reference.log gpurun_out/r2s4_bench_c3.log gpurun_out/r2s4_bench_c2.log; do tail -c 400 $f; echo; done
