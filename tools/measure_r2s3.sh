#!/bin/bash
# Round-2 end-of-work measurements on one GPU (outputs gpurun_out/r2s3_*): the GPU suite, smoke, the default bench
# (C4) and its reference arm, a C4 launch list of 2 fine-tune ticks, and --set full captures of the pairs attention
# (C4 prefill / FT tiles) and the C4 decode attention.
set -x
python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2s3_gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke.log 2>&1
python bench.py > gpurun_out/r2s3_bench_c4.log 2>&1
python bench.py --impl reference > gpurun_out/r2s3_bench_c4_reference.log 2>&1
P="ncu --profile-from-start off --clock-control none"
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s3_c4_launches.csv \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 2 > gpurun_out/r2s3_launch_c4.log 2>&1
$P --set full --import-source on -k regex:attn_fa2 -s 4 -c 1 -o gpurun_out/r2s3_fa2_c4 \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2s3_ncu_fa2.log 2>&1
$P --set full --import-source on -k regex:gemm_tc2 -s 20 -c 1 -o gpurun_out/r2s3_gemm2_c4 \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2s3_ncu_gemm2.log 2>&1
tail -2 gpurun_out/r2s3_gpu_tests.log; tail -1 gpurun_out/r2s3_smoke.log
