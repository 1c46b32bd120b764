set -x
python bench.py > gpurun_out/r1s3_bench_c2.log 2>&1
python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r1s3_bench_c3.log 2>&1
python bench.py --workload c4 --no-cpu-baseline > gpurun_out/r1s3_bench_c4.log 2>&1
python bench.py --impl reference > gpurun_out/r1s3_bench_c2_reference.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r1s3_c2_launches.csv python tools/profile_tick.py --steps 8 > gpurun_out/r1s3_launch_run.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r1s3_c4_launches.csv python tools/profile_tick.py --workload c4 --steps 2 > gpurun_out/r1s3_launch_c4.log 2>&1
