#!/bin/bash
# final-code extras: C4 with 8 LoRA tenants; the N>1 bench path rehearsed with two ranks on one GPU (gloo grads)
set -x
python bench.py --lora-tenants 8 > gpurun_out/r2s5g_bench_c4_lora8.log 2>&1
MACE_ONE_GPU=1 MACE_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --workload c2 --steps 10 --warmup 3 \
  --no-cpu-baseline > gpurun_out/r2s5g_2rank_rehearsal_c2.log 2>&1
tail -c 300 gpurun_out/r2s5g_bench_c4_lora8.log; echo; tail -c 300 gpurun_out/r2s5g_2rank_rehearsal_c2.log
