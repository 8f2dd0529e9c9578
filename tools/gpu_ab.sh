mkdir -p gpurun_out
sum() { python -c "import json,sys; d=json.loads([l for l in open('$1') if l.startswith('{')][-1]); F=d['config']['frames_per_step']; print('$2', round(d['value']), {k:round(v*1000/F,1) for k,v in d['stages_ms_per_step'].items()})" >> gpurun_out/z_sum.txt 2>&1; }
cp exp_libs/libfgs_${FINAL}.so paper_2310_08528_b200/libfgs.so
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/z_pytest.log 2>&1; echo rc=$? >> gpurun_out/z_pytest.log
for V in $VARIANTS; do
  cp exp_libs/libfgs_$V.so paper_2310_08528_b200/libfgs.so
  for c in $CFGS; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/z_${V}_$c.log 2>&1; sum gpurun_out/z_${V}_$c.log "$V $c"; done
  for N in $NS; do timeout 300 python bench.py --n $N --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/z_${V}_n$N.log 2>&1; sum gpurun_out/z_${V}_n$N.log "$V n$N"; done
done
cp exp_libs/libfgs_${FINAL}.so paper_2310_08528_b200/libfgs.so
