#!/bin/bash
# Round measurements on one GPU: bench lines (C2 with cpu_baseline, C3, C4, C2 reference arm) and ncu launch
# lists of 8 C2 / 2 C4 ticks. Usage: bash tools/measure_round.sh TAG  (outputs gpurun_out/TAG_*)
T=${1:-round}
set -x
python bench.py > gpurun_out/${T}_bench_c2.log 2>&1
python bench.py --workload c3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1
python bench.py --workload c4 --no-cpu-baseline > gpurun_out/${T}_bench_c4.log 2>&1
python bench.py --impl reference > gpurun_out/${T}_bench_c2_reference.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_c2_launches.csv python tools/profile_tick.py --steps 8 > gpurun_out/${T}_launch_run.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_c4_launches.csv python tools/profile_tick.py --workload c4 --steps 2 > gpurun_out/${T}_launch_c4.log 2>&1
