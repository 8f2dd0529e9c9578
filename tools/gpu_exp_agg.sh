mkdir -p gpurun_out
for V in ${VARIANTS:-base agg}; do
  cp exp_libs/libfgs_$V.so paper_2310_08528_b200/libfgs.so
  for c in dnerf neu3d scaling; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/y_${V}_$c.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/y_${V}_$c.log').read().strip().splitlines()[-1]); F=d['config']['frames_per_step']; print('$V $c', round(d['value']), {k:round(v*1000/F,1) for k,v in d['stages_ms_per_step'].items() if k in ('preprocess','duplicate')})" >> gpurun_out/y_sum.txt
  done
done
cp exp_libs/libfgs_${FINAL:-base}.so paper_2310_08528_b200/libfgs.so
[ -n "$PYT" ] && timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/y_pytest.log 2>&1; echo rc=$? >> gpurun_out/y_pytest.log
