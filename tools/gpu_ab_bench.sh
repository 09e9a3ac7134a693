mkdir -p gpurun_out
timeout 300 python tools/geglu_bench.py > gpurun_out/geglu_bench.log 2>&1
: > gpurun_out/ab_bench.log
for v in "X=1" "DP_FUSED_GEGLU_BWD=0" "DP_FLIP_BATCH=0" "DP_FUSED_GEGLU=0"; do
  echo "== $v" >> gpurun_out/ab_bench.log
  env $v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | cut -c1-200 >> gpurun_out/ab_bench.log
done
