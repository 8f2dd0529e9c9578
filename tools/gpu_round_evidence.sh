#!/bin/bash
# Round-end evidence pass: profile_all (bench, launch list, ncu full), other configs, colour heads, shard mode, reference arm, N sweep.
TAG=${1:-ev}
bash tools/gpu_profile_all.sh ${TAG}
for c in hypernerf neu3d scaling; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_cfg_$c.log 2>&1; done
timeout 600 python bench.py --colour-heads --no-cpu-baseline > gpurun_out/${TAG}_colour.log 2>&1
timeout 600 python bench.py --config scaling --mode shard --no-cpu-baseline > gpurun_out/${TAG}_shard.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_reference.log 2>&1
bash tools/sweep_n.sh ${TAG}
