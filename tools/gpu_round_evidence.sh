#!/bin/bash
# Round-end evidence pass: profile_all (bench, launch list, ncu full), other configs, colour heads, shard mode, reference arm, N sweep.
TAG=${1:-ev}
bash tools/gpu_profile_all.sh ${TAG}
for c in hypernerf neu3d scaling; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_cfg_$c.log 2>&1; done
timeout 600 python bench.py --colour-heads --no-cpu-baseline > gpurun_out/${TAG}_colour.log 2>&1
timeout 600 python bench.py --config scaling --mode shard --no-cpu-baseline > gpurun_out/${TAG}_shard.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_reference.log 2>&1
bash tools/sweep_n.sh ${TAG}
# training side: train-mode benches and ncu captures of the two backward kernels
timeout 900 python bench.py --mode train > gpurun_out/${TAG}_train.log 2>&1
timeout 600 python bench.py --mode train --config neu3d --no-cpu-baseline > gpurun_out/${TAG}_train_neu3d.log 2>&1
timeout 600 python tools/backward_report.py > gpurun_out/${TAG}_bwd_report.json 2> gpurun_out/${TAG}_bwd_report.err
python tools/bwd_one.py dnerf 3 > gpurun_out/${TAG}_bwd_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"blend_backward|deform_backward|preprocess_backward" \
    -s 6 -c 3 -o gpurun_out/${TAG}_backward -f python tools/bwd_one.py dnerf 3 > gpurun_out/${TAG}_bwd_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_backward.ncu-rep > gpurun_out/${TAG}_backward.summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/${TAG}_backward.ncu-rep 30 > gpurun_out/${TAG}_backward.lines.txt 2>&1
[ "${KEEP_REPS:-0}" = "1" ] || rm -f gpurun_out/${TAG}_backward.ncu-rep
