# bias-gradient fusions: kernel tests, c2 parity, bench A/B (env switches off = old path)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "geglu_bwd_bias or row_bias_bwd_conv or bias_grad" > gpurun_out/fuse_tests.log 2>&1; echo rc=$? >> gpurun_out/fuse_tests.log
timeout -s KILL 900 python -m pytest tests/test_c2_parity_gpu.py tests/test_optimizer_overlap_gpu.py -q -x > gpurun_out/fuse_parity.log 2>&1; echo rc=$? >> gpurun_out/fuse_parity.log
: > gpurun_out/ab_bench.log
for r in 1 2; do
for v in "X=1" "DP_GEGLU_BIAS_DB=0 DP_ROW_BIAS_DB=0"; do
  echo "== $v" >> gpurun_out/ab_bench.log
  env $v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | cut -c1-200 >> gpurun_out/ab_bench.log
done
done
