#!/bin/bash
# Round-2 final evidence pass (r02e): GPU suite (normal + checked build), smoke, bench, then the full
# round evidence (profile_all: launch list + ncu --set full of every forward kernel; other configs, colour
# heads, shard mode, reference arm, N sweep, training side, backward report and ncu).
TAG=${1:-r02e}
bash tools/gpu_check.sh ${TAG}
FGS_LIB=checked timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_checked_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_checked_pytest.log
bash tools/gpu_round_evidence.sh ${TAG}
