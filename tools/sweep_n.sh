#!/bin/bash
# frames/s vs number of Gaussians at 800x800 (D distributions, 20 frames per step).
TAG=${1:-sweep}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for N in 10000 30000 100000 300000 1000000 3000000; do
  timeout 600 python bench.py --n $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' >> gpurun_out/${TAG}_sweep.jsonl
done
