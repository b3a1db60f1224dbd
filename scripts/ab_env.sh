#!/bin/bash
# A/B of one env toggle on one box: bench lines with the default / the toggle / the default.
#   bash scripts/ab_env.sh TAG ENV_ASSIGNMENT workload...
tag=$1; toggle=$2; shift 2
for w in "$@"; do
  timeout 300 python bench.py --workload $w > gpurun_out/ab_${tag}_${w}_on1.log 2>&1
  env $toggle timeout 300 python bench.py --workload $w > gpurun_out/ab_${tag}_${w}_off.log 2>&1
  timeout 300 python bench.py --workload $w > gpurun_out/ab_${tag}_${w}_on2.log 2>&1
done
