#!/bin/bash
# Round-2 session-5 final measurements on one GPU (outputs gpurun_out/r2s5f_*): GPU suite, smoke, default bench (C4)
# and its reference arm, C3 / C2 lines, C3 tick split, the C4 launch list, ncu --set full of the tcgen05 decode
# attention (C4 tick, C3 tick, microbench hd 128).
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s5f_gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s5f_smoke.log 2>&1
python bench.py > gpurun_out/r2s5f_bench_c4.log 2>&1
python bench.py --impl reference > gpurun_out/r2s5f_bench_c4_reference.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s5f_bench_c3.log 2>&1
python bench.py --workload c2 > gpurun_out/r2s5f_bench_c2.log 2>&1
python tools/tick_split.py c3 > gpurun_out/r2s5f_tick_split_c3.log 2>&1
P="ncu --profile-from-start off --clock-control none"
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s5f_c4_launches.csv \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 2 > gpurun_out/r2s5f_launch_c4.log 2>&1
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s5f_c3_launches.csv \
   python tools/profile_tick.py --workload c3 --steps 4 > gpurun_out/r2s5f_launch_c3.log 2>&1
$P --set full --import-source on -k regex:attn_decode_tc -s 4 -c 1 -o gpurun_out/r2s5f_dtc_c4 \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 1 > gpurun_out/r2s5f_ncu_dtc_c4.log 2>&1
$P --set full --import-source on -k regex:attn_decode_tc -s 4 -c 1 -o gpurun_out/r2s5f_dtc_c3 \
   python tools/profile_tick.py --workload c3 --steps 2 > gpurun_out/r2s5f_ncu_dtc_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode_tc -s 3 -c 1 \
    -o gpurun_out/r2s5f_dtc128_micro python tools/decode_bench.py 2 128 32 8 256 1500 > gpurun_out/r2s5f_ncu_dtc128.log 2>&1
tail -2 gpurun_out/r2s5f_gpu_tests.log; tail -1 gpurun_out/r2s5f_smoke.log
for f in c4 c4_reference c3 c2; do tail -c 300 gpurun_out/r2s5f_bench_$f.log; echo; done
tail -3 gpurun_out/r2s5f_tick_split_c3.log; ls -la gpurun_out/r2s5f_*
