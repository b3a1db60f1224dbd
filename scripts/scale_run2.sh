#!/bin/bash
# N = 2 / 4 GPT and N = 4 Wide-ResNet lines on one 4-GPU box (driver launch form)
run() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
  --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n "$@"; }
run 2 > gpurun_out/scale2_gpt_n2.log 2>&1
run 4 > gpurun_out/scale2_gpt_n4.log 2>&1
run 4 --workload moe > gpurun_out/scale2_moe_n4.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_4gpu.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_4gpu.log
