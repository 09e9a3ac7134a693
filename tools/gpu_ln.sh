mkdir -p gpurun_out
: > gpurun_out/ln_bench.log
for v in "DP_LN_GROUPS=1" "DP_LNQ_FULLGRID=1" "DP_LN_GROUPS=0"; do
  echo "== $v" >> gpurun_out/ln_bench.log
  env $v timeout 300 python tools/ln_bench.py >> gpurun_out/ln_bench.log 2>&1
done
