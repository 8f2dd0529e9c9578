#!/bin/bash
# A/B of prebuilt library variants exp_libs/libfgs_<V>.so (e.g. FGS_NVCC_EXTRA="-D..." builds): the
# per-stage bench numbers of several configs for each.  Usage (from gpurun): bash tools/gpu_variants.sh V1 V2 ...
# CONFIGS env: "config:frames[:n] ..." (default the D/N3/H/S benches with short batches for H and S).
mkdir -p gpurun_out
cp paper_2310_08528_b200/libfgs.so /tmp/libfgs_orig.so
CONFIGS=${CONFIGS:-"dnerf:20 neu3d:8 hypernerf:10 scaling:8"}
for V in "$@"; do
  cp exp_libs/libfgs_$V.so paper_2310_08528_b200/libfgs.so; touch paper_2310_08528_b200/libfgs.so
  for CF in $CONFIGS; do
    IFS=: read -r c f n <<< "$CF"
    NARG=""; TAGN=""
    if [ -n "$n" ]; then NARG="--n $n"; TAGN="$n"; fi
    timeout 300 python bench.py --config $c --frames $f $NARG --no-e2e --no-cpu-baseline --steps 10 --warmup 3 \
      > gpurun_out/v_${V}${TAGN:+n$TAGN}_$c.log 2>&1
    echo "$V $c $n rc=$?"
  done
done
cp /tmp/libfgs_orig.so paper_2310_08528_b200/libfgs.so; touch paper_2310_08528_b200/libfgs.so
