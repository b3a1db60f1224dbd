#!/bin/bash
# A/B of the TMA-store GEMM epilogue on one box: bench lines with it on / off / on
set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests3.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests3.log
for w in gpt moe; do
  timeout 300 python bench.py --workload $w > gpurun_out/ab_${w}_on1.log 2>&1
  MPEXEC_GEMM_NO_C_TMA=1 timeout 300 python bench.py --workload $w > gpurun_out/ab_${w}_off.log 2>&1
  timeout 300 python bench.py --workload $w > gpurun_out/ab_${w}_on2.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
