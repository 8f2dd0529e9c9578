#!/bin/bash
# Like tools/gpu_exp.sh for arbitrary configs: bash tools/gpu_exp_cfg.sh "cfg1 cfg2" V1 V2 ...
mkdir -p gpurun_out
CFGS=$1; shift
for V in "$@"; do
  cp paper_2310_08528_b200/build/exp/libfgs_$V.so paper_2310_08528_b200/libfgs.so; touch paper_2310_08528_b200/libfgs.so
  for c in $CFGS; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/x_${V}_$c.log 2>&1
  done
done
