#!/bin/bash
# Run the D and N3 benches for prebuilt library variants (paper_2310_08528_b200/build/exp/libfgs_<V>.so,
# e.g. built with FGS_NVCC_EXTRA="-DFGS_EXP_NOEPI"): deform-stage decomposition experiments.
# Usage (from gpurun): bash tools/gpu_exp.sh V1 V2 ...
mkdir -p gpurun_out
for V in "$@"; do
  cp paper_2310_08528_b200/build/exp/libfgs_$V.so paper_2310_08528_b200/libfgs.so; touch paper_2310_08528_b200/libfgs.so
  for c in dnerf neu3d; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/x_${V}_$c.log 2>&1
  done
done
