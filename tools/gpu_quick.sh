#!/bin/bash
# Quick GPU iteration: deform/frames parity subset + frame-mode bench of D, N3, H.  Usage: bash tools/gpu_quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "deform or frames or colour" > gpurun_out/${TAG}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_pytest.log
for c in dnerf neu3d hypernerf; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_$c.log 2>&1; done
tail -2 gpurun_out/${TAG}_pytest.log
