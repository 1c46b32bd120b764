#!/bin/bash
# Round-2 session-5 final (after the SwiGLU epilogue fix) measurements on one GPU (outputs gpurun_out/r2s5g_*): GPU suite, smoke, default bench (C4)
# and its reference arm, C3 / C2 lines, C3 tick split, C4 / C3 / C2 launch lists.
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s5g_gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s5g_smoke.log 2>&1
python bench.py > gpurun_out/r2s5g_bench_c4.log 2>&1
python bench.py --impl reference > gpurun_out/r2s5g_bench_c4_reference.log 2>&1
python bench.py --workload c3 > gpurun_out/r2s5g_bench_c3.log 2>&1
python bench.py --workload c2 > gpurun_out/r2s5g_bench_c2.log 2>&1
python tools/tick_split.py c3 > gpurun_out/r2s5g_tick_split_c3.log 2>&1
P="ncu --profile-from-start off --clock-control none"
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s5g_c4_launches.csv \
   python tools/profile_tick.py --workload c4 --skip 8 --steps 2 > gpurun_out/r2s5g_launch_c4.log 2>&1
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s5g_c3_launches.csv \
   python tools/profile_tick.py --workload c3 --steps 4 > gpurun_out/r2s5g_launch_c3.log 2>&1
$P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2s5g_c2_launches.csv \
   python tools/profile_tick.py --workload c2 --steps 8 > gpurun_out/r2s5g_launch_c2.log 2>&1
tail -2 gpurun_out/r2s5g_gpu_tests.log; tail -1 gpurun_out/r2s5g_smoke.log
for f in c4 c4_reference c3 c2; do tail -c 300 gpurun_out/r2s5g_bench_$f.log; echo; done
tail -3 gpurun_out/r2s5g_tick_split_c3.log; ls -la gpurun_out/r2s5g_*
