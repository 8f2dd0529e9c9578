#!/bin/bash
# Full evidence pass on one GPU: bench, ncu launch list, ncu --set full of every kernel of the step.
TAG=${1:-prof}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
for KS in blend_kernel:2 deform_tc3_kernel:2 preprocess_kernel:2 tile_sort_kernel:2 duplicate_kernel:2 tile_scan_kernel:2; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K} -s ${S} -c 1 \
     -o gpurun_out/${TAG}_${K} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
     > gpurun_out/${TAG}_${K}_ncu.log 2>&1
  echo "$K rc=$?"
  # reports are tens of MB (gpurun brings back <= 64 MiB): keep their text summaries
  python tools/ncu_summary.py gpurun_out/${TAG}_${K}.ncu-rep > gpurun_out/${TAG}_${K}.summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/${TAG}_${K}.ncu-rep 30 > gpurun_out/${TAG}_${K}.lines.txt 2>&1
  [ "${KEEP_REPS:-0}" = "1" ] || rm -f gpurun_out/${TAG}_${K}.ncu-rep
done
