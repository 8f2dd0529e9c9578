#!/bin/bash
# ncu --set full captures of the top kernels (one launch each) of the default bench workload.
# Usage: bash tools/gpu_ncu_full.sh TAG "kernel:skip kernel:skip ..."
TAG=${1:-r1}
LIST=${2:-"blend_kernel:2 deform_tc3_kernel:2 tile_sort_kernel:2 preprocess_kernel:2"}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for KS in $LIST; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K} -s ${S} -c 1 \
     -o gpurun_out/${TAG}_${K} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
     > gpurun_out/${TAG}_${K}_ncu.log 2>&1
  echo "$K rc=$?"
done
